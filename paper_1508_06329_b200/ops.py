"""Device-level operations: thin wrappers over the C ABI on torch tensors.

Every function here launches CUDA work on the current torch stream and
returns device tensors; the reference-shaped entry points in ``search``,
``peo`` and ``parallel`` convert to numpy / 1-based types at the edge.
PyTorch only allocates memory and provides the stream.
"""

from __future__ import annotations

import numpy as np

from . import _native
from ._native import check, lib, ptr, stream_ptr
from .device import DeviceRows

U64_MAX = (1 << 64) - 1


def _i32(torch, n, dev):
    return torch.empty(max(n, 1), dtype=torch.int32, device=dev)


def _ws(torch, nbytes, dev):
    return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=dev)


def lexbfs(rows: DeviceRows, tie_rule: int = _native.TIE_ASCENDING, seed: int = 0, m: int = -1, stream=None,
           want_parent: bool = False):
    """LexBFS on device rows -> (order, pos[, parent]) int32 device tensors.

    ``m`` is the edge count (chooses the engine); -1 lets the library count it.
    """
    torch = _native.require_cuda()
    n, dev = rows.n, rows.data.device
    order, pos, parent = _i32(torch, n, dev), _i32(torch, n, dev), _i32(torch, n, dev)
    if n:
        mm = _edge_count(rows, m, stream)
        ws = _ws(torch, lib.chordal_dense_workspace_bytes(n, mm), dev)
        check(
            lib.chordal_lexbfs_dense(rows.ptr, n, rows.stride, mm, tie_rule, seed & U64_MAX, ptr(order), ptr(pos),
                                     ptr(parent) if want_parent else None, ptr(ws), ws.numel(), stream_ptr(stream)),
            "chordal_lexbfs_dense",
        )
    if want_parent:
        return order[:n], pos[:n], parent[:n]
    return order[:n], pos[:n]


def lexbfs_certify(rows: DeviceRows, order, m: int = -1, stream=None) -> tuple[int, int]:
    """Replay LexBFS with the pivots forced to ``order`` (int32 device tensor) ->
    (first step whose pivot is not in the maximum-label class, first step whose
    pivot is not the LOWEST_INDEX choice), -1 for none (chordal_lexbfs_certify_dense)."""
    torch = _native.require_cuda()
    n, dev = rows.n, rows.data.device
    status = torch.empty(2, dtype=torch.int32, device=dev)
    ws = _ws(torch, lib.chordal_lexbfs_certify_workspace_bytes(n), dev)
    mm = m if m >= 0 else rows.m
    check(lib.chordal_lexbfs_certify_dense(rows.ptr, n, rows.stride, mm, ptr(order) if n else None, ptr(status),
                                           ptr(ws), ws.numel(), stream_ptr(stream)), "chordal_lexbfs_certify_dense")
    s = status.cpu().tolist()
    return int(s[0]), int(s[1])


def _edge_count(rows: DeviceRows, m: int, stream=None) -> int:
    """The edge count the dense entry points need: only graphs above the
    shared-memory engine's limit (n > 32768, CSR route) need it; the others
    pass 0 and skip the counting pass and its host synchronisation."""
    if m >= 0:
        return m
    if rows.m >= 0:
        return rows.m
    if rows.n <= _native.DENSE_LEXBFS_MAX_N:
        return 0
    return count_edges(rows, stream)


def csr_from_rows(rows: DeviceRows, stream=None):
    """Device CSR (indptr int64[n+1], indices int32[2m], ascending rows) of device rows."""
    torch = _native.require_cuda()
    dev = rows.data.device
    indptr = torch.empty(rows.n + 1, dtype=torch.int64, device=dev)
    check(lib.chordal_dense_to_csr(rows.ptr, rows.n, rows.stride, ptr(indptr), None, stream_ptr(stream)),
          "chordal_dense_to_csr")
    nnz = int(indptr[rows.n].item())
    rows.m = nnz // 2
    indices = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
    check(lib.chordal_dense_to_csr(rows.ptr, rows.n, rows.stride, ptr(indptr), ptr(indices), stream_ptr(stream)),
          "chordal_dense_to_csr")
    return indptr, indices[:nnz]


def count_edges(rows: DeviceRows, stream=None) -> int:
    """Edge count of device rows (one popcount pass + a 8-byte read-back)."""
    torch = _native.require_cuda()
    indptr = torch.empty(rows.n + 1, dtype=torch.int64, device=rows.data.device)
    check(lib.chordal_dense_to_csr(rows.ptr, rows.n, rows.stride, ptr(indptr), None, stream_ptr(stream)),
          "chordal_dense_to_csr")
    rows.m = int(indptr[rows.n].item()) // 2
    return rows.m


def permute(rows: DeviceRows, perm0: np.ndarray, stream=None) -> DeviceRows:
    """Relabelled copy: row r, bit s = rows[perm0[r]][perm0[s]]."""
    torch = _native.require_cuda()
    p = torch.as_tensor(np.ascontiguousarray(perm0, dtype=np.int32)).to(rows.data.device)
    out = torch.empty_like(rows.data)
    check(lib.chordal_permute_dense(rows.ptr, rows.n, rows.stride, ptr(p), ptr(out), stream_ptr(stream)),
          "chordal_permute_dense")
    return DeviceRows(rows.n, rows.stride, out, rows.m)


def positions(order, stream=None):
    torch = _native.require_cuda()
    n = int(order.numel())
    pos = _i32(torch, n, order.device)
    if n:
        check(lib.chordal_positions(ptr(order), n, ptr(pos), stream_ptr(stream)), "chordal_positions")
    return pos[:n]


def peo(rows: DeviceRows, order, pos, parent=None, stream=None):
    """PEO check -> witness int32[3] device tensor ((-1,-1,-1) when a PEO)."""
    torch = _native.require_cuda()
    key = torch.empty(1, dtype=torch.int64, device=rows.data.device)
    wit = torch.empty(4, dtype=torch.int32, device=rows.data.device)
    n = rows.n
    check(
        lib.chordal_peo_dense(rows.ptr, n, rows.stride, ptr(order) if n else None, ptr(pos) if n else None,
                              ptr(parent) if (n and parent is not None) else None, ptr(key), ptr(wit),
                              stream_ptr(stream)),
        "chordal_peo_dense",
    )
    return wit[:3]


def peo_key(rows: DeviceRows, order, pos, v_begin: int, v_end: int, key, parent=None, stream=None):
    """Accumulate the minimum violation key of v in [v_begin, v_end) into ``key`` (int64[1])."""
    check(
        lib.chordal_peo_dense_key(rows.ptr, rows.n, rows.stride, ptr(order), ptr(pos),
                                  ptr(parent) if parent is not None else None, v_begin, v_end, ptr(key),
                                  stream_ptr(stream)),
        "chordal_peo_dense_key",
    )


def key_init(key, stream=None):
    check(lib.chordal_key_init(ptr(key), stream_ptr(stream)), "chordal_key_init")


def peo_witness(rows: DeviceRows, pos, key, stream=None):
    torch = _native.require_cuda()
    wit = torch.empty(4, dtype=torch.int32, device=rows.data.device)
    check(
        lib.chordal_peo_dense_witness(rows.ptr, rows.n, rows.stride, ptr(pos) if rows.n else None, ptr(key),
                                      ptr(wit), stream_ptr(stream)),
        "chordal_peo_dense_witness",
    )
    return wit[:3]


def is_chordal(rows: DeviceRows, tie_rule: int = _native.TIE_ASCENDING, seed: int = 0, m: int = -1, stream=None,
               ws=None):
    """Fused pipeline -> (order, pos, witness) device tensors."""
    torch = _native.require_cuda()
    n, dev = rows.n, rows.data.device
    order, pos = _i32(torch, n, dev), _i32(torch, n, dev)
    wit = torch.empty(4, dtype=torch.int32, device=dev)
    mm = _edge_count(rows, m, stream)
    if ws is None:
        ws = _ws(torch, lib.chordal_dense_workspace_bytes(n, max(mm, 0)), dev)
    check(
        lib.chordal_is_chordal_dense(rows.ptr, n, rows.stride, mm, tie_rule, seed & U64_MAX, ptr(order), ptr(pos),
                                     ptr(ws), ws.numel(), ptr(wit), stream_ptr(stream)),
        "chordal_is_chordal_dense",
    )
    return order[:n], pos[:n], wit[:3]


def dense_workspace(n: int, m: int, device="cuda"):
    torch = _native.require_cuda()
    return _ws(torch, lib.chordal_dense_workspace_bytes(n, m), device)


# ---------------------------------------------------------------- CSR ------


def lexbfs_csr(indptr, indices, n: int, tie_rule: int = _native.TIE_ASCENDING, seed: int = 0, stream=None,
               m: int | None = None):
    """LexBFS on device CSR -> (order, pos, parent) int32 device tensors."""
    torch = _native.require_cuda()
    dev = indptr.device
    order, pos, parent = _i32(torch, n, dev), _i32(torch, n, dev), _i32(torch, n, dev)
    if n:
        if m is None:
            m = int(indices.numel()) // 2
        ws = _ws(torch, lib.chordal_lexbfs_csr_workspace_bytes(n, m), dev)
        if indices.numel() == 0:  # edgeless: the ABI wants a real pointer
            indices = torch.zeros(1, dtype=torch.int32, device=dev)
        check(
            lib.chordal_lexbfs_csr(ptr(indptr), ptr(indices), n, m, tie_rule, seed & U64_MAX, ptr(order), ptr(pos),
                                   ptr(parent), ptr(ws), ws.numel(), stream_ptr(stream)),
            "chordal_lexbfs_csr",
        )
    return order[:n], pos[:n], parent[:n]


def peo_csr_workspace(n: int, device):
    torch = _native.require_cuda()
    return _ws(torch, lib.chordal_peo_csr_workspace_bytes(n), device)


def peo_csr(indptr, indices, n: int, pos, parent=None, stream=None, ws=None):
    torch = _native.require_cuda()
    dev = indptr.device
    key = torch.empty(1, dtype=torch.int64, device=dev)
    wit = torch.empty(4, dtype=torch.int32, device=dev)
    ws = ws if ws is not None else peo_csr_workspace(n, dev)
    check(
        lib.chordal_peo_csr(ptr(indptr), ptr(indices), n, ptr(pos) if n else None,
                            ptr(parent) if (n and parent is not None) else None, ptr(key), ptr(wit),
                            ptr(ws), ws.numel(), stream_ptr(stream)),
        "chordal_peo_csr",
    )
    return wit[:3]


def peo_csr_key(indptr, indices, n: int, pos, v_begin: int, v_end: int, key, parent=None, stream=None, ws=None):
    ws = ws if ws is not None else peo_csr_workspace(n, indptr.device)
    check(
        lib.chordal_peo_csr_key(ptr(indptr), ptr(indices), n, ptr(pos), ptr(parent) if parent is not None else None,
                                v_begin, v_end, ptr(key), ptr(ws), ws.numel(), stream_ptr(stream)),
        "chordal_peo_csr_key",
    )


def peo_csr_witness(indptr, indices, n: int, pos, key, stream=None):
    torch = _native.require_cuda()
    wit = torch.empty(4, dtype=torch.int32, device=indptr.device)
    check(lib.chordal_peo_csr_witness(ptr(indptr), ptr(indices), n, ptr(pos) if n else None, ptr(key), ptr(wit),
                                      stream_ptr(stream)), "chordal_peo_csr_witness")
    return wit[:3]


def left_dense(rows: DeviceRows, order, pos, want_rows: bool = True, stream=None):
    """(LN rows uint8[n, stride] or None, parent, |LN|, deg) int32 device tensors
    (left_neighborhoods, graph.py:284-302)."""
    torch = _native.require_cuda()
    n, dev = rows.n, rows.data.device
    ln = torch.empty((n, rows.stride), dtype=torch.uint8, device=dev) if want_rows else None
    parent, ln_size, deg = (_i32(torch, n, dev) for _ in range(3))
    check(lib.chordal_left_dense(rows.ptr, n, rows.stride, ptr(order), ptr(pos), ptr(ln) if want_rows else None,
                                 ptr(parent), ptr(ln_size), ptr(deg), stream_ptr(stream)), "chordal_left_dense")
    return ln, parent, ln_size, deg


def left_csr(indptr, indices, n: int, order, pos, stream=None):
    """(parent, |LN|) int32 device tensors of a CSR graph under an ordering."""
    torch = _native.require_cuda()
    dev = indptr.device
    parent, ln_size = _i32(torch, n, dev), _i32(torch, n, dev)
    check(lib.chordal_left_csr(ptr(indptr), ptr(indices), n, ptr(order), ptr(pos), ptr(parent), ptr(ln_size),
                               stream_ptr(stream)), "chordal_left_csr")
    return parent, ln_size


def dense_to_csr(rows: DeviceRows, stream=None):
    """Packed rows -> (indptr int64[n+1], indices int32[2m]) on the device."""
    torch = _native.require_cuda()
    n, dev = rows.n, rows.data.device
    indptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    check(lib.chordal_dense_to_csr(rows.ptr, n, rows.stride, ptr(indptr), None, stream_ptr(stream)),
          "chordal_dense_to_csr")
    nnz = int(indptr[n].item())
    indices = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
    check(lib.chordal_dense_to_csr(rows.ptr, n, rows.stride, ptr(indptr), ptr(indices), stream_ptr(stream)),
          "chordal_dense_to_csr")
    return indptr, indices[:nnz]


# -------------------------------------------------------------- batches ----


def is_chordal_batch(adj, n: int, stride: int, stream=None):
    """Batched pipeline on adj uint8[B, n, stride] -> (orders int32[B,n], witness int32[B,3])."""
    torch = _native.require_cuda()
    B = int(adj.shape[0])
    orders = torch.empty((max(B, 1), max(n, 1)), dtype=torch.int32, device=adj.device)
    # empty graphs are chordal: witness (-1, -1, -1) (the library writes it for n == 0 too)
    wit = torch.empty((max(B, 1), 3), dtype=torch.int32, device=adj.device)
    if B:
        check(
            lib.chordal_is_chordal_batch(ptr(adj), B, n, stride, ptr(orders), ptr(wit), stream_ptr(stream)),
            "chordal_is_chordal_batch",
        )
    return orders[:B, :n], wit[:B]


def gen_dense_random(adj, n: int, stride: int, p: float, seed0: int, seed_step: int = 1, stream=None):
    """Fill adj uint8[B, n, stride] with gen_dense_random(n, p, seed0 + b*seed_step)."""
    B = int(adj.shape[0])
    if B and n:
        check(
            lib.chordal_gen_dense_random(ptr(adj), B, n, stride, float(p), int(seed0), int(seed_step),
                                         stream_ptr(stream)),
            "chordal_gen_dense_random",
        )
    return adj


def gen_chordal_random(adj, n: int, stride: int, k: int, seed0: int, seed_step: int = 1, stream=None):
    """Fill adj uint8[B, n, stride] with gen_chordal_random(n, k, seed0 + b*seed_step)."""
    torch = _native.require_cuda()
    B = int(adj.shape[0])
    if B and n:
        nbytes = int(lib.chordal_gen_chordal_random_scratch_bytes(B, n, k))
        scratch = torch.empty(max(nbytes, 4), dtype=torch.uint8, device=adj.device)
        check(
            lib.chordal_gen_chordal_random(ptr(adj), B, n, stride, int(k), int(seed0), int(seed_step), ptr(scratch),
                                           nbytes, stream_ptr(stream)),
            "chordal_gen_chordal_random",
        )
    return adj


def edges_to_dense(u0, v0, n: int, stride: int, out=None, stream=None):
    """0-based endpoint arrays (host or device) -> device rows uint8[n, stride]."""
    torch = _native.require_cuda()
    u = torch.as_tensor(np.asarray(u0, dtype=np.int32) if not hasattr(u0, "device") else u0).to("cuda", torch.int32)
    v = torch.as_tensor(np.asarray(v0, dtype=np.int32) if not hasattr(v0, "device") else v0).to("cuda", torch.int32)
    if out is None:
        out = torch.empty((max(n, 1), stride), dtype=torch.uint8, device="cuda")
    check(lib.chordal_edges_to_dense(ptr(u), ptr(v), int(u.numel()), ptr(out), n, stride, stream_ptr(stream)),
          "chordal_edges_to_dense")
    return out[:n]


def witness_tuple(w) -> tuple[int, int, int] | None:
    """Device witness tensor -> 0-based (v, p, z) or None."""
    a = w.cpu().numpy() if hasattr(w, "cpu") else np.asarray(w)
    return None if int(a[0]) < 0 else (int(a[0]), int(a[1]), int(a[2]))


# ------------------------------------------------------- other orderings ----


def mcs(rows: DeviceRows, seeded: bool = False, seed: int = 0, stream=None):
    """Maximum cardinality search on device rows -> (order, pos) int32 device tensors."""
    torch = _native.require_cuda()
    n, dev = rows.n, rows.data.device
    order, pos = _i32(torch, n, dev), _i32(torch, n, dev)
    if n:
        check(lib.chordal_mcs_dense(rows.ptr, n, rows.stride, int(bool(seeded)), seed & U64_MAX, ptr(order),
                                    ptr(pos), stream_ptr(stream)), "chordal_mcs_dense")
    return order[:n], pos[:n]


def bfs_csr(indptr, indices, n: int, seeded: bool = False, seed: int = 0, stream=None):
    """Breadth-first order on device CSR -> (order, pos) int32 device tensors."""
    torch = _native.require_cuda()
    dev = indptr.device
    order, pos = _i32(torch, n, dev), _i32(torch, n, dev)
    if n:
        if indices.numel() == 0:
            indices = torch.zeros(1, dtype=torch.int32, device=dev)
        wsb = int(lib.chordal_bfs_csr_workspace_bytes(n))
        ws = _ws(torch, wsb, dev) if wsb else None
        check(lib.chordal_bfs_csr(ptr(indptr), ptr(indices), n, int(bool(seeded)), seed & U64_MAX, ptr(order),
                                  ptr(pos), ptr(ws) if ws is not None else None, wsb, stream_ptr(stream)),
              "chordal_bfs_csr")
    return order[:n], pos[:n]


def bfs_dense(rows: DeviceRows, seeded: bool = False, seed: int = 0, stream=None):
    """Breadth-first order on device rows (word-parallel) -> (order, pos) int32 device tensors."""
    torch = _native.require_cuda()
    n, dev = rows.n, rows.data.device
    order, pos = _i32(torch, n, dev), _i32(torch, n, dev)
    if n:
        check(lib.chordal_bfs_dense(rows.ptr, n, rows.stride, int(bool(seeded)), seed & U64_MAX, ptr(order),
                                    ptr(pos), stream_ptr(stream)), "chordal_bfs_dense")
    return order[:n], pos[:n]
