"""Multi-process (gloo, world_size 2) tests of the sharding protocols on CPU.

The per-rank compute is an oracle-backed stand-in for the CUDA backend (test
infrastructure); what is under test is the host protocol of
paper_1508_06329_b200.distributed: shard bounds, order/parent broadcast, the
MIN all-reduce of the violation key, witness resolution and batch gathers.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1508_06329_b200.distributed import (
    batch_shard,
    count_chordal,
    gather_batch,
    shard_bounds,
    sharded_is_chordal,
)


def test_shard_bounds_cover_exactly():
    for total in (0, 1, 7, 512, 65536, 1000003):
        for world in (1, 2, 3, 4, 8):
            parts = [shard_bounds(total, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [h - l for l, h in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


class OracleBackend:
    """CPU stand-in for CudaBackend (same contract, oracle arithmetic)."""

    def device(self):
        return torch.device("cpu")

    @staticmethod
    def _rows(g):
        return np.unpackbits(np.asarray(g._packed), axis=1, bitorder="little", count=g.n).astype(bool)

    def lexbfs(self, g):
        import oracle

        order = oracle.lexbfs_partition(g._packed, g.n)
        return torch.from_numpy(order.astype(np.int32)), None, None

    def positions(self, order):
        pos = torch.empty_like(order)
        pos[order.long()] = torch.arange(order.numel(), dtype=order.dtype)
        return pos

    def peo_key(self, g, order, pos, parent, lo, hi):
        rows, p = self._rows(g), pos.numpy()
        best = (1 << 64) - 1
        for v in range(lo, hi):
            left = np.flatnonzero(rows[v] & (p < p[v]))
            if left.size == 0:
                continue
            par = int(left[np.argmax(p[left])])
            stray = rows[v] & ~rows[par] & (p < p[par])
            stray[par] = False
            if stray.any():
                best = min(best, (par << 32) | v)
        return torch.tensor([best - (1 << 64) if best >= 1 << 63 else best], dtype=torch.int64)

    def witness(self, g, pos, key):
        k = int(key.item())
        if k == -1:
            return None
        par, v = k >> 32, k & 0xFFFFFFFF
        rows, p = self._rows(g), pos.numpy()
        stray = rows[v] & ~rows[par] & (p < p[par])
        stray[par] = False
        return v, par, int(np.flatnonzero(stray)[0])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1508_06329_b200.generate import gen_chordal_random, gen_dense_random, remove_first_chord

        out = {}
        for name, g in (("chordal", gen_chordal_random(300, 5, 1)),
                        ("nonchordal", remove_first_chord(gen_chordal_random(300, 5, 2))[0]),
                        ("dense", gen_dense_random(120, 0.5, 3))):
            v = sharded_is_chordal(g, backend=OracleBackend())
            out[name] = (v.chordal, None if v.witness is None else (v.witness.v, v.witness.p, v.witness.z),
                         None if v.peo is None else v.peo.order0.tolist())
        lo, hi = batch_shard(10)
        wl = torch.tensor([[-1, -1, -1] if (lo + i) % 3 else [lo + i, 0, 0] for i in range(hi - lo)],
                          dtype=torch.int32)
        out["gather"] = gather_batch(wl, 10)
        out["count"] = count_chordal(wl)
        results[rank] = out
    finally:
        dist.destroy_process_group()


def test_row_sharded_peo_and_batch_gather_gloo():
    import oracle
    from paper_1508_06329_b200.generate import gen_chordal_random, gen_dense_random, remove_first_chord

    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    expect = {}
    for name, g in (("chordal", gen_chordal_random(300, 5, 1)),
                    ("nonchordal", remove_first_chord(gen_chordal_random(300, 5, 2))[0]),
                    ("dense", gen_dense_random(120, 0.5, 3))):
        ok, order, w = oracle.is_chordal(g._packed, g.n)
        expect[name] = (ok, None if w is None else (w[0] + 1, w[1] + 1, w[2] + 1), order.tolist() if ok else None)
    for r in range(world):
        for name in expect:
            assert results[r][name] == expect[name], (r, name)
        assert results[r]["count"] == sum(1 for b in range(10) if b % 3)
    g0 = results[0]["gather"]
    assert g0.shape == (10, 3)
    assert [int(x) for x in g0[:, 0]] == [b if b % 3 == 0 else -1 for b in range(10)]
    assert results[1]["gather"] is None


def _gpu_worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)  # one B200 in this environment: both ranks share it
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1508_06329_b200.csr import CSRGraph
        from paper_1508_06329_b200.generate import gen_chordal_random, gen_dense_random, remove_first_chord

        out = {}
        graphs = {"c1": gen_chordal_random(1000, 8, 0), "c1x": remove_first_chord(gen_chordal_random(1000, 8, 0))[0],
                  "dense": gen_dense_random(700, 0.5, 4),
                  "csr": CSRGraph.from_dense(remove_first_chord(gen_chordal_random(3000, 6, 5))[0])}
        for name, g in graphs.items():
            v = sharded_is_chordal(g)  # the CUDA backend
            out[name] = (v.chordal, None if v.witness is None else (v.witness.v, v.witness.p, v.witness.z))
        results[rank] = out
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_row_sharded_peo_cuda_backend_two_ranks():
    import oracle
    from paper_1508_06329_b200.generate import gen_chordal_random, gen_dense_random, remove_first_chord

    world = 2
    results = mp.Manager().dict()
    mp.spawn(_gpu_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    graphs = {"c1": gen_chordal_random(1000, 8, 0), "c1x": remove_first_chord(gen_chordal_random(1000, 8, 0))[0],
              "dense": gen_dense_random(700, 0.5, 4),
              "csr": remove_first_chord(gen_chordal_random(3000, 6, 5))[0]}
    for name, g in graphs.items():
        ok, _, w = oracle.is_chordal(g._packed, g.n)
        exp = (ok, None if w is None else (w[0] + 1, w[1] + 1, w[2] + 1))
        assert results[0][name] == exp and results[1][name] == exp, name


@pytest.mark.gpu
def test_nccl_c_abi_single_rank_matches_oracle():
    """chordal_is_chordal_{dense,csr}_nccl through a one-rank NCCL communicator
    (torch.cuda.nccl; this environment has one GPU): the broadcast / shard /
    MIN all-reduce protocol of the C ABI gives the oracle's verdicts, orders and
    witnesses."""
    import ctypes
    import glob

    import numpy as np

    import oracle
    from paper_1508_06329_b200.csr import CSRGraph
    from paper_1508_06329_b200.distributed import sharded_is_chordal_nccl
    from paper_1508_06329_b200.generate import chordal_random_edges, gen_chordal_random, gen_dense_random, \
        remove_first_chord

    torch.cuda.set_device(0)
    torch.zeros(1, device="cuda")  # CUDA context up before NCCL
    # the NCCL torch ships (the library our entry points resolve by soname)
    libs = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "nccl", "lib", "libnccl.so*"))
    nccl = ctypes.CDLL(libs[0] if libs else "libnccl.so.2", mode=ctypes.RTLD_GLOBAL)

    class UniqueId(ctypes.Structure):
        _fields_ = [("internal", ctypes.c_char * 128)]

    uid = UniqueId()
    assert nccl.ncclGetUniqueId(ctypes.byref(uid)) == 0
    comm_p = ctypes.c_void_p()
    nccl.ncclCommInitRank.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, UniqueId, ctypes.c_int]
    assert nccl.ncclCommInitRank(ctypes.byref(comm_p), 1, uid, 0) == 0
    comm = int(comm_p.value)
    graphs = {"c1": gen_chordal_random(1000, 8, 0), "c1x": remove_first_chord(gen_chordal_random(1000, 8, 0))[0],
              "dense": gen_dense_random(2500, 0.5, 4), "chordal3k": gen_chordal_random(3000, 30, 1)}
    for name, g in graphs.items():
        ok, order, w = oracle.is_chordal(g._packed, g.n)
        for gg in (g, CSRGraph.from_dense(g)):
            v = sharded_is_chordal_nccl(gg, comm)
            assert v.chordal == ok, name
            if ok:
                assert v.peo.order0.tolist() == order.tolist(), name
            else:
                assert (v.witness.v - 1, v.witness.p - 1, v.witness.z - 1) == tuple(w), name
    n = 40000  # the global-state slot engine, parents broadcast from the search
    u, vv = chordal_random_edges(n, 4, 3)
    big = CSRGraph.from_edges0(n, u, vv)
    v = sharded_is_chordal_nccl(big, comm)
    order = oracle.lexbfs_partition_csr(big.indptr, big.indices, n)
    assert v.chordal and np.array_equal(v.peo.order0, order)
    nccl.ncclCommDestroy.argtypes = [ctypes.c_void_p]
    nccl.ncclCommDestroy(ctypes.c_void_p(comm))
