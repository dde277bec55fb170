"""Engine dispatch shared by the reference-shaped entry points.

Dense inputs (``_packed`` rows) go through chordal_lexbfs_dense /
chordal_is_chordal_dense (the shared-memory touched-segment engine for
n <= 32768, the CSR slot engine above); CSR inputs through the CSR kernels.  Everything returns host
numpy arrays (0-based) at the end -- the only device->host copies of a call.
"""

from __future__ import annotations

import numpy as np

from . import _native, ops
from .csr import device_csr, is_csr
from .device import device_rows
from .graph import VertexOrdering


def lexbfs(g, tie_rule: int, seed: int = 0) -> VertexOrdering:
    n = int(g.n)
    if n == 0:
        return VertexOrdering(())
    if is_csr(g):
        ip, ix = device_csr(g)
        order, pos, _ = ops.lexbfs_csr(ip, ix, n, tie_rule, seed)
    else:
        order, pos = ops.lexbfs(device_rows(g), tie_rule, seed)
    return VertexOrdering._trusted(order.cpu().numpy(), pos.cpu().numpy())


def lexbfs_linked_seeded(g, tie_rule: int, seed: int) -> VertexOrdering:
    """The seeded *linked* LexBFS variants (TIE_SEEDED_PARTITION / _LABELS) run on
    the CSR slot engine (dense inputs are converted to CSR on the device)."""
    n = int(g.n)
    if n == 0:
        return VertexOrdering(())
    if is_csr(g):
        ip, ix = device_csr(g)
    else:
        ip, ix = ops.csr_from_rows(device_rows(g))
    order, pos, _ = ops.lexbfs_csr(ip, ix, n, tie_rule, seed, m=int(ix.numel()) // 2)
    return VertexOrdering._trusted(order.cpu().numpy(), pos.cpu().numpy())


def certify_lexbfs(g, o: VertexOrdering) -> tuple[int, int]:
    """Device certificate of ``o`` as a LexBFS order of ``g`` (ops.lexbfs_certify):
    0-based (first step whose pivot lacks the maximum label, first step that is
    not the LOWEST_INDEX choice), -1 for none.  CSR inputs are expanded to
    bit rows on the device; the replay engine holds n <= 32768."""
    torch = _native.require_cuda()
    n = int(g.n)
    if n == 0:
        return -1, -1
    if n > _native.DENSE_LEXBFS_MAX_N:
        from .errors import GraphTooLarge

        raise GraphTooLarge(f"the device LexBFS certificate (debug / audit) holds n <= "
                            f"{_native.DENSE_LEXBFS_MAX_N}, got n={n}")
    if is_csr(g):
        from .graph import device_stride
        from .device import DeviceRows

        ip, ix = device_csr(g)
        u = torch.repeat_interleave(torch.arange(n, dtype=torch.int32, device=ip.device), ip[1:] - ip[:-1])
        st = device_stride(n)
        rows = DeviceRows(n, st, ops.edges_to_dense(u, ix[: u.numel()], n, st), m=int(ix.numel()) // 2)
    else:
        rows = device_rows(g)
    order = torch.as_tensor(np.ascontiguousarray(o.order0, dtype=np.int32)).to(rows.data.device)
    return ops.lexbfs_certify(rows, order)


def peo_witness(g, o: VertexOrdering):
    """0-based witness of the PEO test of ordering ``o`` (None when a PEO)."""
    torch = _native.require_cuda()
    if is_csr(g):
        ip, ix = device_csr(g)
        order = torch.as_tensor(np.ascontiguousarray(o.order0, dtype=np.int32)).to(ip.device)
        return ops.witness_tuple(ops.peo_csr(ip, ix, int(g.n), ops.positions(order)))
    rows = device_rows(g)
    order = torch.as_tensor(np.ascontiguousarray(o.order0, dtype=np.int32)).to(rows.data.device)
    return ops.witness_tuple(ops.peo(rows, order, ops.positions(order)))


def left_arrays(g, o: VertexOrdering, want_rows: bool):
    """Host arrays of the left-neighbourhood kernels (csrc/left.cu) under ``o``:
    (LN rows uint8[n, ceil(n/8)] or None, parent int32[n] (-1: none), |LN| int32[n],
    deg int64[n]).  LN rows exist for dense inputs only."""
    torch = _native.require_cuda()
    n = int(g.n)
    if is_csr(g):
        ip, ix = device_csr(g)
        order = torch.as_tensor(np.ascontiguousarray(o.order0, dtype=np.int32)).to(ip.device)
        parent, ln_size = ops.left_csr(ip, ix, n, order, ops.positions(order))
        deg = np.diff(ip.cpu().numpy())
        return None, parent[:n].cpu().numpy(), ln_size[:n].cpu().numpy(), deg
    rows = device_rows(g)
    order = torch.as_tensor(np.ascontiguousarray(o.order0, dtype=np.int32)).to(rows.data.device)
    ln, parent, ln_size, deg = ops.left_dense(rows, order, ops.positions(order), want_rows)
    ln_h = ln[:, : (n + 7) // 8].cpu().numpy() if want_rows else None
    return ln_h, parent[:n].cpu().numpy(), ln_size[:n].cpu().numpy(), deg[:n].cpu().numpy().astype(np.int64)


def is_chordal(g, tie_rule: int, seed: int = 0):
    """LexBFS + PEO test on the device: (VertexOrdering, 0-based witness or None)."""
    n = int(g.n)
    if n == 0:
        return VertexOrdering(()), None
    if is_csr(g):
        ip, ix = device_csr(g)
        order, pos, parent = ops.lexbfs_csr(ip, ix, n, tie_rule, seed)
        wit = ops.peo_csr(ip, ix, n, pos, parent)
    else:
        order, pos, wit = ops.is_chordal(device_rows(g), tie_rule, seed)
    w0 = ops.witness_tuple(wit)
    return VertexOrdering._trusted(order.cpu().numpy(), pos.cpu().numpy()), w0


def mcs_order(g, seeded: bool, seed: int) -> VertexOrdering:
    n = int(g.n)
    if n == 0:
        return VertexOrdering(())
    if is_csr(g):
        raise NotImplementedError("mcs_order runs on dense rows (n <= 65535); pass a Graph")
    order, pos = ops.mcs(device_rows(g), seeded, seed)
    return VertexOrdering._trusted(order.cpu().numpy(), pos.cpu().numpy())


def bfs_order(g, seeded: bool, seed: int) -> VertexOrdering:
    n = int(g.n)
    if n == 0:
        return VertexOrdering(())
    if is_csr(g):
        ip, ix = device_csr(g)
        order, pos = ops.bfs_csr(ip, ix, n, seeded, seed)
    elif n <= 65535:  # dense rows: word-parallel fresh-neighbour masks
        order, pos = ops.bfs_dense(device_rows(g), seeded, seed)
    else:
        ip, ix = ops.csr_from_rows(device_rows(g))
        order, pos = ops.bfs_csr(ip, ix, n, seeded, seed)
    return VertexOrdering._trusted(order.cpu().numpy(), pos.cpu().numpy())
