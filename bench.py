"""Benchmark of the chordality test (LexBFS + PEO check) on B200.

Headline (BASELINE.json metric "chordality-test ms/graph (N=32k dense) and
graphs/sec batched at 1/2/4/8 B200 vs CPU"):
  value      graphs/s of configuration 4 -- 65,536 independent graphs of 512
             vertices (seed s: gen_dense_random(512, 0.5, s) if s is even, else
             gen_chordal_random(512, 8, s)), sharded over the ranks by
             contiguous seed ranges (strong scaling: the total is fixed).  One
             step = one is_chordal pass over the whole batch, inputs resident
             in HBM (2 GiB at N=1 > 126 MB L2, so no flush is needed).
  e2e        the same metric through the host-buffer C-ABI entry point
             chordal_is_chordal_batch_host (pinned host graphs in, orders +
             witnesses out, copies inside the timed region).
  dense32k   ms/graph of configuration 3 (N=32768: chordal k=1024, its
             chord-removed twin, and G(32768, 0.5)), plus configurations 1-2, on
             rank 0 -- device-resident ("algo") and host-buffer ("total").
Inputs are synthetic but bit-identical to the reference generators (drawn
on the GPU by csrc/gen.cu).  --impl reference times the reference algorithm
(the C port in oracle/, all host threads) on a bounded sample.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DATA = "synthetic (the reference generators replayed bit-exact)"
METRIC = "chordality-test ms/graph (N=32k dense) and graphs/sec batched at 1/2/4/8 B200 vs CPU"
N512, STRIDE512, K512 = 512, 64, 8
TOTAL_GRAPHS = 65536
BYTES_PER_GRAPH = N512 * STRIDE512 + 4 * N512 + 12  # adjacency read + order + witness written


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--graphs", type=int, default=TOTAL_GRAPHS)
    ap.add_argument("--no-secondary", action="store_true", help="skip the N=32k / N=8k / N=1k lines")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks --


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------- utils --


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks() -> tuple[dict, str]:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def shard(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous seed range of `rank`: the ranges tile [0, total) exactly for any world."""
    return total * rank // world, total * (rank + 1) // world


def build_batch(lo: int, hi: int, device):
    """Graphs of seeds [lo, hi) in seed order, drawn on the GPU (bit-exact)."""
    import torch

    from paper_1508_06329_b200.generate import gen_chordal_random_device, gen_dense_random_device

    B = hi - lo
    adj = torch.empty((B, N512, STRIDE512), dtype=torch.uint8, device=device)
    ev = range(lo + (lo % 2), hi, 2)
    od = range(lo + 1 - (lo % 2), hi, 2)
    if len(ev):
        adj[(ev.start - lo)::2] = gen_dense_random_device(N512, 0.5, ev, stride=STRIDE512)
    if len(od):
        adj[(od.start - lo)::2] = gen_chordal_random_device(N512, K512, od, stride=STRIDE512)
    torch.cuda.synchronize()
    return adj


def reduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum_ints(vals: list[int], world: int) -> list[int]:
    if world == 1:
        return list(vals)
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor(vals, dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [int(x) for x in t.tolist()]


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


# ------------------------------------------------------------- cpu baseline --


PARITY_SAMPLE = 8192  # graphs of each rank's shard checked against the oracle every run


def check_batch_parity(adj_host: np.ndarray, orders, wit, seed_lo: int, time_it: bool) -> dict:
    """The oracle (C port of the reference's is_chordal, oracle/) on the first
    PARITY_SAMPLE graphs of this rank's shard -- the graphs the timed loop ran --
    compared bit for bit with the GPU's orders, verdicts and witnesses; raises on
    any difference.  When time_it, the same run is the cpu_baseline (all host
    threads; rank 0 at N=1)."""
    import oracle

    S = min(len(adj_host), PARITY_SAMPLE)
    threads = oracle.max_threads()
    # the inputs themselves: the GPU generator's graphs against the oracle's C
    # restatement of the reference generators (sha-pinned to the reference)
    ref_adj = oracle.gen_config4_batch(seed_lo, S, N512, 0.5, K512, STRIDE512, nthreads=threads)
    if not np.array_equal(ref_adj, adj_host[:S]):
        raise SystemExit(f"PARITY FAILURE on configuration 4: the device-generated graphs of seeds "
                         f"{seed_lo}..{seed_lo + S - 1} differ from the reference generators")
    del ref_adj
    t0 = time.perf_counter()
    verdict, o_ref, w_ref = oracle.is_chordal_batch(adj_host[:S], N512, nthreads=threads)
    dt = time.perf_counter() - t0
    o_gpu = orders[:S].cpu().numpy()
    w_gpu = wit[:S].cpu().numpy()
    bad_w = np.nonzero((w_gpu != w_ref).any(axis=1))[0]
    # orders are compared where the reference returns one: every graph's LexBFS order
    bad_o = np.nonzero((o_gpu != o_ref).any(axis=1))[0]
    if len(bad_w) or len(bad_o) or not np.array_equal(w_gpu[:, 0] < 0, verdict):
        first = int((list(bad_w) + list(bad_o) + [0])[0])
        raise SystemExit(f"PARITY FAILURE on configuration 4: {len(bad_o)} orders and {len(bad_w)} witnesses of "
                         f"the first {S} graphs differ from the oracle (first: seed {seed_lo + first})")
    out = {"graphs": S, "seeds": [seed_lo, seed_lo + S - 1], "inputs_equal": True, "orders_equal": True, "witnesses_equal": True,
           "verdicts_equal": True, "chordal": int(verdict.sum())}
    if time_it:
        out["cpu_baseline"] = {"value": S / dt, "unit": "graphs/s", "cores": threads, "kind": "port",
                               "sample": f"first {S} graphs (seeds {seed_lo}..{seed_lo + S - 1}) of configuration 4, "
                                         f"oracle/ C port of is_chordal (PartitionList LexBFS + list PEO) per graph, "
                                         f"{threads} host threads"}
    return out


# --------------------------------------------------------------- secondary --


# ~10 ms of device spin queued ahead of a timed region, so that a kernel time is
# not stretched by the host's own call overhead (ctypes, argument checks) or by
# host scheduling noise on the box; it ends before the start event fires.
SPIN_CYCLES = 20_000_000


def time_events(fn, reps: int = 3, warm: int = 1) -> float:
    import torch

    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(SPIN_CYCLES)  # device busy while the host enqueues: no launch gaps inside s..e
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def single_graph_lines(with_cpu: bool) -> dict:
    """Configurations 1-3 on rank 0: per-graph ms, LexBFS ns/step, PEO roofline."""
    import torch

    import paper_1508_06329_b200 as P
    from paper_1508_06329_b200 import _native, ops
    from paper_1508_06329_b200.device import DeviceRows
    from paper_1508_06329_b200.generate import (
        chordal_random_edges,
        gen_dense_random_device,
        remove_first_chord,
    )
    from paper_1508_06329_b200.graph import device_stride

    peaks, _ = measured_peaks()
    out = {}

    def rows_from_edges(n, k, seed):
        u, v = chordal_random_edges(n, k, seed)
        return DeviceRows(n, device_stride(n), ops.edges_to_dense(u, v, n, device_stride(n)))

    cpu = {}

    def cpu_leg(name, packed, n, w_gpu, order_gpu):
        """The oracle C port of is_chordal (PartitionList LexBFS + list PEO, 1 core)
        on the same graph, and the GPU result checked against it."""
        import oracle

        packed = np.ascontiguousarray(packed)
        t0 = time.perf_counter()
        o_ref = oracle.lexbfs_partition(packed, n)
        t1 = time.perf_counter()
        ok, w_ref = oracle.is_peo(packed, n, o_ref)
        t2 = time.perf_counter()
        same = bool(np.array_equal(o_ref, order_gpu)) and (w_ref == w_gpu)
        if not same:
            raise SystemExit(f"PARITY FAILURE on {name}: GPU order/witness differ from the oracle")
        cpu[name] = {"ms_per_graph": (t2 - t0) * 1e3, "lexbfs_ms": (t1 - t0) * 1e3, "peo_ms": (t2 - t1) * 1e3,
                     "cores": 1, "kind": "port", "same_order_and_witness": same}

    def measure(name, rows: DeviceRows, host_packed=None):
        n = rows.n
        if rows.m < 0:  # Graph.m, as the public API passes it (picks the engine's thread count)
            ops.count_edges(rows)
        lex = time_events(lambda: ops.lexbfs(rows))
        order, pos, parent = ops.lexbfs(rows, want_parent=True)
        # PEO check as the pipeline runs it (parents handed over by LexBFS), and
        # standalone is_peo on the same order (parents searched by the kernel)
        peo = time_events(lambda: ops.peo(rows, order, pos, parent))
        peo_search = time_events(lambda: ops.peo(rows, order, pos))
        full = time_events(lambda: ops.is_chordal(rows))
        _, _, wit = ops.is_chordal(rows)
        w = ops.witness_tuple(wit)
        rec = {"n": n, "ms_per_graph": full, "lexbfs_ms": lex, "lexbfs_ns_per_step": lex * 1e6 / n,
               "peo_ms": peo, "peo_parent_search_ms": peo_search, "chordal": w is None,
               "witness": None if w is None else [w[0] + 1, w[1] + 1, w[2] + 1]}
        peo_bytes = 2 * n * rows.stride + 12 * n
        if w is None:  # a chordal graph: every vertex's row and its parent's row are read
            rec["peo_roofline"] = {"bound": "hbm", "achieved_gbs": peo_bytes / (peo * 1e-3) / 1e9,
                                   "frac": peo_bytes / (peo * 1e-3) / 1e9 / peaks["hbm_gbs"],
                                   "algorithmic_bytes": peo_bytes}
        else:  # violators found early let the other warps skip their rows: no fraction
            rec["peo_roofline"] = {"bound": "hbm", "frac": None, "algorithmic_bytes_full_check": peo_bytes,
                                   "full_check_equivalent_gbs": peo_bytes / (peo * 1e-3) / 1e9,
                                   "note": "non-chordal: warps whose witness key cannot beat the current "
                                           "minimum skip their rows, so a full check's bytes are not all read"}
        if host_packed is not None:
            hp = np.ascontiguousarray(host_packed)
            order_h = np.empty(n, dtype=np.int32)
            wit_h = np.empty(3, dtype=np.int32)
            flag = ctypes.c_int32()

            m_ = int(rows.m)
            wsb = int(_native.lib.chordal_dense_host_workspace_bytes(n, m_))
            ws_t = torch.empty(wsb + 256, dtype=torch.uint8, device="cuda")
            wp = (ws_t.data_ptr() + 255) & ~255

            def e2e():
                rc = _native.lib.chordal_is_chordal_dense_host_ws(hp.ctypes.data, n, hp.shape[1], m_, 0, 0,
                                                                  order_h.ctypes.data, wit_h.ctypes.data,
                                                                  ctypes.byref(flag), wp, wsb)
                _native.check(rc, "chordal_is_chordal_dense_host_ws")

            e2e()
            t0 = time.perf_counter()
            for _ in range(3):
                e2e()
            rec["total_ms_host_buffers"] = (time.perf_counter() - t0) / 3 * 1e3
        out[name] = rec
        if with_cpu:
            packed = host_packed if host_packed is not None else rows.data[:, : (n + 7) // 8].cpu().numpy()
            cpu_leg(name, packed, n, w, order.cpu().numpy())
            rec["cpu_baseline"] = cpu[name]

    # configuration 3 (N = 32768)
    r3 = rows_from_edges(32768, 1024, 0)
    measure("c3_chordal_k1024", r3)
    g3 = P.Graph._from_packed(32768, r3.data[:, :4096].cpu().numpy())
    h3, _ = remove_first_chord(g3)
    r3n = DeviceRows(32768, 4096, torch.from_numpy(np.array(h3._packed)).cuda())
    measure("c3_nonchordal", r3n, h3._packed)
    d3 = gen_dense_random_device(32768, 0.5, 0)[0]
    measure("c3_dense_p0.5", DeviceRows(32768, 4096, d3))
    del d3, r3n
    # configuration 2 (N = 8192)
    d2 = gen_dense_random_device(8192, 0.5, 0)[0]
    measure("c2_dense_p0.5", DeviceRows(8192, 1024, d2), d2.cpu().numpy())
    measure("c2_chordal_k8", rows_from_edges(8192, 8, 0))
    # configuration 1 (N = 1000)
    r1 = rows_from_edges(1000, 8, 0)
    g1 = P.Graph._from_packed(1000, r1.data[:, :125].cpu().numpy())
    h1, _ = remove_first_chord(g1)
    measure("c1_chordal_k8", r1, g1._packed)
    measure("c1_nonchordal", DeviceRows(1000, 128, torch.from_numpy(
        np.pad(np.array(h1._packed), ((0, 0), (0, 3)))).cuda()), h1._packed)
    # configuration 5 (N = 10^6 CSR, chordal k = 8): drawn on the GPU, LexBFS + PEO
    from paper_1508_06329_b200.generate import gen_chordal_random_csr_device

    t0 = time.perf_counter()
    ip5, ix5 = gen_chordal_random_csr_device(1_000_000, 8, 0)
    torch.cuda.synchronize()
    gen5 = time.perf_counter() - t0
    n5 = 1_000_000
    lex5 = time_events(lambda: ops.lexbfs_csr(ip5, ix5, n5), reps=1, warm=1)
    o5, p5, par5 = ops.lexbfs_csr(ip5, ix5, n5)
    peo5 = time_events(lambda: ops.peo_csr(ip5, ix5, n5, p5, par5), reps=3)
    w5 = ops.witness_tuple(ops.peo_csr(ip5, ix5, n5, p5, par5))
    nnz = int(ix5.numel())
    peo5_bytes = 2 * 4 * nnz + 8 * (n5 + 1) + 12 * n5  # both rows' index lists + indptr + pos/parent/order
    out["c5_csr_chordal_k8_n1e6"] = {
        "n": n5, "m": nnz // 2, "ms_per_graph": lex5 + peo5, "lexbfs_ms": lex5,
        "lexbfs_ns_per_step": lex5 * 1e6 / n5, "peo_ms": peo5, "chordal": w5 is None,
        "device_generation_s": gen5,
        "peo_roofline": {"bound": "hbm", "achieved_gbs": peo5_bytes / (peo5 * 1e-3) / 1e9,
                         "frac": peo5_bytes / (peo5 * 1e-3) / 1e9 / peaks["hbm_gbs"], "algorithmic_bytes": peo5_bytes},
    }
    # the other orderings and the text formats: GPU time beside the
    # oracle's C port of the reference algorithm (1 core) on the same graph
    from paper_1508_06329_b200 import textio
    from paper_1508_06329_b200.generate import gen_dense_random as gen_dense_host

    g2 = gen_dense_host(8192, 0.5, 0, cap=8192)
    rows2 = DeviceRows(8192, device_stride(8192), torch.from_numpy(
        np.pad(np.asarray(g2._packed), ((0, 0), (0, device_stride(8192) - g2._packed.shape[1])))).cuda(), m=g2.m)
    ip2, ix2 = ops.csr_from_rows(rows2)
    mcs_ms = time_events(lambda: ops.mcs(rows2))
    bfs_ms = time_events(lambda: ops.bfs_dense(rows2))
    bfs_csr_ms = time_events(lambda: ops.bfs_csr(ip2, ix2, 8192))
    txt = textio.write_graph_text(g2)
    t0 = time.perf_counter()
    g2b = textio.parse_graph_text(txt, cap=8192)
    parse_s = time.perf_counter() - t0
    assert g2b == g2
    other = {"graph": "gen_dense_random(8192, 0.5, 0)", "m": int(g2.m),
             "mcs_order_ms": mcs_ms, "bfs_order_ms": bfs_ms, "bfs_order_csr_ms": bfs_csr_ms,
             "parse_graph_text": {"bytes": len(txt), "s": parse_s, "MBps": len(txt) / parse_s / 1e6, "threads": 1}}
    if with_cpu:
        import oracle

        t0 = time.perf_counter()
        oracle.other_order(g2._packed, 8192, "mcs")
        t1 = time.perf_counter()
        oracle.other_order(g2._packed, 8192, "bfs")
        t2 = time.perf_counter()
        other["cpu_baseline"] = {"mcs_order_ms": (t1 - t0) * 1e3, "bfs_order_ms": (t2 - t1) * 1e3, "cores": 1,
                                 "kind": "port"}
    out["orders_and_text"] = other
    if with_cpu:
        import oracle

        ip_h, ix_h = ip5.cpu().numpy(), ix5.cpu().numpy()
        t0 = time.perf_counter()
        o_h = oracle.lexbfs_partition_csr(ip_h, ix_h, n5)
        t1 = time.perf_counter()
        oracle.is_peo_csr(ip_h, ix_h, n5, o_h)
        t2 = time.perf_counter()
        cpu["c5_csr_chordal_k8_n1e6"] = {"ms_per_graph": (t2 - t0) * 1e3, "lexbfs_ms": (t1 - t0) * 1e3,
                                         "peo_ms": (t2 - t1) * 1e3, "cores": 1, "kind": "port",
                                         "same_order": bool((o_h == o5.cpu().numpy()).all())}
        if not cpu["c5_csr_chordal_k8_n1e6"]["same_order"]:
            raise SystemExit("PARITY FAILURE on c5: GPU order differs from the oracle")
        out["c5_csr_chordal_k8_n1e6"]["cpu_baseline"] = cpu["c5_csr_chordal_k8_n1e6"]
        out["cpu_baseline"] = cpu
    return out


def row_sharded_lines(rank: int, world: int, reps: int = 5) -> dict:
    """Configurations 5 (CSR N = 10^6) and 3 (dense N = 32768, chord-removed) with the
    PEO check row-sharded over all ranks: LexBFS on rank 0 (replicas
    only -- its per-step chain stays on one GPU), order + parents broadcast, each
    rank tests its contiguous rows, one 8-byte MIN all-reduce of the witness key,
    z resolved locally.  Timed on the device from the broadcast to the witness, max
    over ranks; the per-rank PEO kernel time is reported beside it."""
    import torch
    import torch.distributed as dist

    from paper_1508_06329_b200 import distributed as D
    from paper_1508_06329_b200 import ops
    from paper_1508_06329_b200.device import DeviceRows
    from paper_1508_06329_b200.generate import chordal_random_edges, gen_chordal_random_csr_device
    from paper_1508_06329_b200.graph import device_stride

    nccl = world > 1 and dist.get_backend() == "nccl"
    dev = torch.device("cuda", torch.cuda.current_device())
    out = {}

    def bcast(t):
        if world > 1:
            if nccl:
                dist.broadcast(t, src=0)
            else:
                h = t.cpu()
                dist.broadcast(h, src=0)
                t.copy_(h)

    def allmin(k):
        if world > 1:
            if nccl:
                dist.all_reduce(k, op=dist.ReduceOp.MIN)
            else:
                h = k.cpu()
                dist.all_reduce(h, op=dist.ReduceOp.MIN)
                k.copy_(h)

    def run(name, n, lexbfs, peo_key, witness):
        if rank == 0:
            order, _, parent = lexbfs()
        else:
            order = torch.empty(n, dtype=torch.int32, device=dev)
            parent = torch.empty(n, dtype=torch.int32, device=dev)
        lo, hi = D.shard_bounds(n, rank, world)
        times, kern = [], []
        w0 = None
        for r in range(reps + 1):
            barrier(world)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ka, kb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(SPIN_CYCLES)
            a.record()
            bcast(order)
            bcast(parent)
            pos = ops.positions(order)
            key = torch.empty(1, dtype=torch.int64, device=dev)
            ops.key_init(key)
            ka.record()
            peo_key(order, pos, parent, lo, hi, key)
            kb.record()
            k = D._to_reducible(key, torch)
            allmin(k)
            w0 = witness(pos, D._from_reducible(k, torch))
            b.record()
            torch.cuda.synchronize()
            if r:  # the first pass warms up
                times.append(a.elapsed_time(b))
                kern.append(ka.elapsed_time(kb))
        out[name] = {"n": n, "ranks": world, "rows_per_rank": hi - lo,
                     "peo_step_ms": reduce_max(sum(times) / len(times), world),
                     "peo_kernel_ms_max_rank": reduce_max(sum(kern) / len(kern), world),
                     "chordal": w0 is None, "witness": None if w0 is None else [w0[0] + 1, w0[1] + 1, w0[2] + 1],
                     "timed": "broadcast(order, parent) + positions + row-shard PEO key + MIN all-reduce + z"}

    # configuration 5: CSR, chordal
    n5 = 1_000_000
    ip5, ix5 = gen_chordal_random_csr_device(n5, 8, 0)
    run("c5_csr_chordal_k8_n1e6", n5, lambda: ops.lexbfs_csr(ip5, ix5, n5),
        lambda o, p, par, lo, hi, key: ops.peo_csr_key(ip5, ix5, n5, p, lo, hi, key, par),
        lambda p, key: ops.witness_tuple(ops.peo_csr_witness(ip5, ix5, n5, p, key)))
    del ip5, ix5
    # configuration 3: dense rows, chord-removed copy (witness (2, 3600, 3))
    n3 = 32768
    u, v = chordal_random_edges(n3, 1024, 0)
    keep = ~((u == 1) & (v == 0)) & ~((u == 0) & (v == 1))  # remove_first_chord drops edge (1, 2)
    rows = DeviceRows(n3, device_stride(n3), ops.edges_to_dense(u[keep], v[keep], n3, device_stride(n3)))
    run("c3_nonchordal", n3, lambda: ops.lexbfs(rows, want_parent=True),
        lambda o, p, par, lo, hi, key: ops.peo_key(rows, o, p, lo, hi, key, par),
        lambda p, key: ops.witness_tuple(ops.peo_witness(rows, p, key)))
    return out


# -------------------------------------------------------------------- main --


def config4(graphs: int) -> dict:
    """The workload both arms name (identical dict in both JSON lines)."""
    return {"workload": "config4: 65536 graphs N=512 (even seed gen_dense_random(512,0.5,s), odd seed "
                        "gen_chordal_random(512,8,s)); one step = is_chordal over every graph",
            "graphs": graphs, "n": N512, "l2": "inputs 2 GiB > L2 (126 MB), no flush needed"}


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU implementation of the path -- the
    oracle's C port of is_chordal (PartitionList LexBFS + list PEO test,
    oracle/chordal_oracle.c) -- on all host threads, over the same configuration-4
    graphs as the GPU arm.  Nothing here loads the product package or the GPU:
    the graphs come from the oracle's own C restatement of the reference
    generators (pinned to the reference's sha256 fixtures in the tests).
    Under torchrun only rank 0 works; the other ranks exit 0."""
    if rank != 0:
        return
    import oracle

    threads = oracle.max_threads()
    G = args.graphs
    t0 = time.perf_counter()
    adj = oracle.gen_config4_batch(0, G, N512, 0.5, K512, STRIDE512, nthreads=threads)
    gen_s = time.perf_counter() - t0

    def step():
        return oracle.is_chordal_batch(adj, N512, nthreads=threads)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        verdict, _, _ = step()
    dt = time.perf_counter() - t0
    value = G * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "graphs/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": DATA,
        "config": config4(G),
        "cpu_baseline": {"value": value, "unit": "graphs/s", "cores": threads, "kind": "port",
                         "sample": f"all {G} graphs of configuration 4 per step (seeds 0..{G - 1}), oracle/ C port "
                                   f"of is_chordal (PartitionList LexBFS + list PEO) per graph, {threads} host threads"},
        "e2e": {"value": value, "unit": "graphs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "input_generation_s": gen_s, "chordal_fraction": float(verdict.mean()),
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local):
    import torch

    from paper_1508_06329_b200 import _native, ops

    # one process per GPU; BENCH_DIST_BACKEND=gloo (host collectives, ranks may
    # share a device) exists only to exercise the multi-rank logic on a 1-GPU box
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            # NCCL's init lines (communicator, nRanks, transport) go to stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(backend)
    lo, hi = shard(args.graphs, rank, world)
    B = hi - lo
    adj = build_batch(lo, hi, device)

    def step():
        return ops.is_chordal_batch(adj, N512, STRIDE512)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    barrier(world)
    stream = torch.cuda.current_stream()
    t_s, t_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier(world)
        t_s.record(stream)
        for _ in range(args.steps):
            step()
        t_e.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    t_ms = reduce_max(t_s.elapsed_time(t_e), world)
    ms_per_step = t_ms / args.steps
    value = args.graphs * args.steps / (t_ms * 1e-3)
    # the timed batch's own results: the first PARITY_SAMPLE graphs of the shard are
    # checked bit for bit against the oracle below (the run fails on a mismatch)
    orders, wit = step()
    torch.cuda.synchronize()

    # e2e through the host-buffer C-ABI: pinned graphs in, orders + witnesses out
    host = torch.empty((B, N512, STRIDE512), dtype=torch.uint8, pin_memory=True)
    host.copy_(adj)
    orders_h = torch.empty((B, N512), dtype=torch.int32, pin_memory=True)
    wit_h = torch.empty((B, 3), dtype=torch.int32, pin_memory=True)

    # the public host-buffer API in its repeated-call form: a device workspace
    # allocated once (like a cuDNN/cuBLAS workspace), reused by every call
    wsb = int(_native.lib.chordal_batch_host_workspace_bytes(N512, 8192))
    e2e_ws = torch.empty(wsb + 256, dtype=torch.uint8, device=device)
    ws_ptr = (e2e_ws.data_ptr() + 255) & ~255

    def e2e_step():
        rc = _native.lib.chordal_is_chordal_batch_host_ws(host.data_ptr(), B, N512, STRIDE512, orders_h.data_ptr(),
                                                          wit_h.data_ptr(), 8192, ws_ptr, wsb)
        _native.check(rc, "chordal_is_chordal_batch_host_ws")

    # first calls map the staging buffers and fault in the pinned pages (the first
    # few calls on a fresh box can take 10x longer)
    for _ in range(max(6, args.warmup)):
        e2e_step()
    e2e_steps = max(3, min(args.steps, 10))
    barrier(world)
    t0 = time.perf_counter()
    call_ms = []
    for _ in range(e2e_steps):
        tc = time.perf_counter()
        e2e_step()
        call_ms.append(round(1e3 * (time.perf_counter() - tc), 2))
    e2e_s = reduce_max(time.perf_counter() - t0, world)
    assert torch.equal(wit_h, wit.cpu()) and torch.equal(orders_h, orders.cpu()), "e2e result differs"
    e2e_value = args.graphs * e2e_steps / e2e_s
    # the e2e leg is bound by the host link: compare its H2D rate with a plain
    # pinned-memory copy of the same size class (best of 3, CUDA events)
    probe = host.view(-1)[: min(host.numel(), 512 << 20)]
    dprobe = torch.empty_like(probe, device=device)
    link_best = 0.0
    for _ in range(3):
        ca, cb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ca.record()
        dprobe.copy_(probe, non_blocking=True)
        cb.record()
        cb.synchronize()
        link_best = max(link_best, probe.numel() / (ca.elapsed_time(cb) * 1e-3) / 1e9)
    del dprobe
    h2d_gbs = B * N512 * STRIDE512 * e2e_steps / e2e_s / 1e9

    peaks, peak_kind = measured_peaks()
    achieved = B * BYTES_PER_GRAPH / (ms_per_step * 1e-3) / 1e9
    traffic = None  # DRAM bytes per launch from the committed ncu --set full capture, scaled to this shard
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        t = json.load(open(tpath)).get("batch_chordal_kernel")
        if t:
            traffic = (t["dram_read_bytes"] + t["dram_write_bytes"]) * B / t["graphs_per_launch"]
    # the bound that matters for this kernel: instruction issue (the LexBFS steps are
    # shuffle / shared-memory chains); warp instructions per graph from the same capture
    issue = None
    if os.path.exists(tpath):
        t = json.load(open(tpath)).get("batch_chordal_kernel", {})
        if t.get("warp_instructions"):
            ipg = t["warp_instructions"] / t["graphs_per_launch"]
            import torch as _t

            sms = _t.cuda.get_device_properties(device).multi_processor_count
            peak_issue = sms * 4 * peaks.get("sm_max_mhz", 1965.0) * 1e6  # 4 schedulers x 1 warp-instr/cycle
            ach = value / world * ipg
            issue = {"bound": "issue", "achieved": ach, "peak": peak_issue, "unit": "warp-instr/s",
                     "frac": ach / peak_issue, "warp_instructions_per_graph": ipg,
                     "source": "smsp__inst_executed.sum of the committed ncu capture (profiles/ncu_traffic.json)"}
    line = {
        "metric": METRIC, "value": value, "unit": "graphs/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8", "data": DATA,
        "config": config4(args.graphs),
        "parallelism": f"batch-shard x{world} (contiguous seed ranges)", "graphs_per_rank": B,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                     "algorithmic_bytes_per_launch": B * BYTES_PER_GRAPH,
                     "kernel": "batch_chordal_kernel", "peak_kind": peak_kind,
                     "algorithmic_bytes_per_graph": BYTES_PER_GRAPH},
        "roofline_issue": issue,
        "e2e": {"value": e2e_value, "unit": "graphs/s", "h2d_bytes_per_step": B * N512 * STRIDE512,
                "d2h_bytes_per_step": B * (4 * N512 + 12), "api": "chordal_is_chordal_batch_host_ws",
                "calls_ms": call_ms,
                "link": {"bound": "pcie_h2d", "achieved_gbs": h2d_gbs, "peak_gbs": link_best,
                         "peak_kind": "measured pinned H2D copy, 512 MiB, best of 3", "frac": h2d_gbs / link_best}},
        "gpu_launches": args.steps,
        "clocks": clk.summary(),
    }
    parity = check_batch_parity(host.numpy(), orders, wit, lo, time_it=rank == 0 and world == 1 and not args.no_cpu)
    if "cpu_baseline" in parity:
        line["cpu_baseline"] = parity.pop("cpu_baseline")
    # every rank's verdicts and parity-checked counts, summed over the ranks
    chordal_total, checked_total, graphs_total = reduce_sum_ints(
        [int((wit[:, 0] < 0).sum().item()), parity["graphs"], B], world)
    assert graphs_total == args.graphs, (graphs_total, args.graphs)
    line["chordal_fraction"] = chordal_total / graphs_total
    line["parity"] = dict(parity, ranks=world, graphs_checked_all_ranks=checked_total,
                          chordal_graphs_all_ranks=chordal_total)
    if not args.no_secondary:
        line["row_sharded_peo"] = row_sharded_lines(rank, world)
    if rank == 0 and world == 1 and not args.no_secondary:
        line["single_graph"] = single_graph_lines(with_cpu=not args.no_cpu)
        line["dense32k"] = {k: v["ms_per_graph"] for k, v in line["single_graph"].items() if k.startswith("c3")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
