"""Perfect-elimination-order test and the chordality pipeline on the GPU.

Same surface as ``chordalkit.peo`` (peo.py:26-202): ``is_peo`` returns
``(bool, WitnessTriple | None)`` with the reference's deterministic witness --
the violating pair with the smallest parent p, then the smallest child v,
then the smallest z (peo.py:81-85, 126-145) -- and ``is_chordal`` returns a
``ChordalityVerdict``.  Both run ``csrc/peo_dense.cu`` (and the LexBFS kernel)
through libchordal_b200.so; the ``method=`` strings of the reference are
accepted for drop-in compatibility and validated the same way, but every
method runs the same CUDA path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native, ops, pipeline
from .errors import InvalidOrdering
from .graph import VertexOrdering, as_ordering
from .search import LOWEST_INDEX, TieBreak, lexbfs_labels, lexbfs_partition

_ARRAY_MIN_N = 1024


@dataclass(frozen=True)
class WitnessTriple:
    """z and p are left neighbours of v, p the latest, z not adjacent to p (peo.py:26-45)."""

    v: int
    p: int
    z: int

    def verify(self, g, ordering) -> bool:
        o = as_ordering(ordering)
        has = _has_edge(g)
        pos = o.pi_inv
        return (
            has(self.v, self.p)
            and has(self.v, self.z)
            and not has(self.p, self.z)
            and pos(self.z) < pos(self.p) < pos(self.v)
        )


def _has_edge(g):
    if hasattr(g, "has_edge"):
        return g.has_edge
    packed = g._packed

    def has(u: int, v: int) -> bool:
        return bool((packed[u - 1, (v - 1) >> 3] >> ((v - 1) & 7)) & 1)

    return has


@dataclass
class ScanStats:
    """List-element reads of the reference's 4-scan test (peo.py:48-56).

    The GPU check does not scan lists; when a ``ScanStats`` is passed, the
    read count the reference's list method would have made on the same input
    is reconstructed from the device's verdict (see ``_list_scan_reads``).
    """

    reads: int = 0
    budget: int = 0

    def within_budget(self) -> bool:
        return self.reads <= self.budget


@dataclass(frozen=True)
class ChordalityVerdict:
    chordal: bool
    peo: VertexOrdering | None = None
    witness: WitnessTriple | None = None

    def __post_init__(self):
        if self.chordal and (self.peo is None or self.witness is not None):
            raise ValueError("chordal verdict must carry a PEO and no witness")
        if not self.chordal and (self.witness is None or self.peo is not None):
            raise ValueError("non-chordal verdict must carry a witness and no PEO")


def _device_order(o: VertexOrdering, device):
    torch = _native.require_cuda()
    order = torch.as_tensor(np.ascontiguousarray(o.order0, dtype=np.int32)).to(device)
    return order, ops.positions(order)


def _witness(w0) -> WitnessTriple | None:
    return None if w0 is None else WitnessTriple(w0[0] + 1, w0[1] + 1, w0[2] + 1)


def is_peo(g, ordering, *, stats: ScanStats | None = None, method: str = "auto"):
    """Test whether ``ordering`` is a perfect elimination order of ``g`` (peo.py:72-97)."""
    o = as_ordering(ordering)
    if o.n != g.n:
        raise InvalidOrdering(f"ordering covers {o.n} vertices, graph has {g.n}")
    if method not in ("auto", "array", "lists"):
        raise ValueError(f"unknown method {method!r}")
    if g.n == 0:
        if stats is not None:
            stats.reads, stats.budget = 0, 0
        return True, None
    w0 = pipeline.peo_witness(g, o)
    if stats is not None:
        stats.reads = _list_scan_reads(g, o, w0)
        stats.budget = 8 * int(g.m)
    return (w0 is None), _witness(w0)


def _row0(g, u: int) -> np.ndarray:
    """Sorted 0-based neighbours of vertex u (one row, host side)."""
    if hasattr(g, "_packed"):
        return np.flatnonzero(np.unpackbits(np.asarray(g._packed)[u], bitorder="little", count=int(g.n)))
    if hasattr(g, "indptr") and hasattr(g, "indices"):
        ip = np.asarray(g.indptr)
        return np.asarray(g.indices)[ip[u] : ip[u + 1]].astype(np.int64)
    return np.asarray(sorted(g.adjacency_lists0()[u]), dtype=np.int64)


def _list_scan_reads(g, o: VertexOrdering, w0) -> int:
    """Reads the reference's list scan (peo.py:100-149) performs on this input.

    Instrumentation only (the verdict comes from the device).  Scan 1 reads
    every adjacency entry; scans 2-4 read, per parent x in ascending order,
    ln[x] twice, adj[x] once and ln[y] of each child y -- up to the witness,
    where the scan stops.  deg, |ln| and the parents come from the device
    (csrc/left.cu), so the count costs O(n) on the host plus the two rows of
    the witness pair, for dense and CSR inputs alike.
    """
    n = int(g.n)
    _, parent, ln_size, deg = pipeline.left_arrays(g, o, want_rows=False)
    ln_size = ln_size.astype(np.int64)
    has = parent >= 0
    child_ln = np.bincount(parent[has], weights=ln_size[has], minlength=n).astype(np.int64)
    reads = int(deg.sum())
    if w0 is None:
        return reads + int((2 * ln_size + deg + child_ln).sum())
    v, p, z = w0
    reads += int((2 * ln_size[:p] + deg[:p] + child_ln[:p]).sum())
    reads += int(ln_size[p])
    nbrs = _row0(g, p)
    upto = nbrs[nbrs <= v]
    reads += int(upto.size)
    before = upto[(upto < v) & (parent[upto] == p)]
    reads += int(ln_size[before].sum())
    nv = _row0(g, v)
    lny = nv[o.pos0[nv] < o.pos0[v]]
    reads += int(np.searchsorted(lny, z) + 1)
    return reads


def is_chordal(g, algo: str = "partition", tie_break: TieBreak = LOWEST_INDEX, *,
               method: str = "auto") -> ChordalityVerdict:
    """LexBFS then the PEO test on its output (peo.py:177-202), fused on the GPU."""
    if method not in ("auto", "reference", "array"):
        raise ValueError(f"unknown method {method!r}")
    if algo not in ("partition", "labels"):
        raise ValueError(f"unknown LexBFS variant {algo!r}")
    n = int(g.n)
    if n == 0:
        return ChordalityVerdict(True, peo=VertexOrdering(()))
    if tie_break.seed is not None:
        lex_method = "linked" if method == "reference" else method
        fn = lexbfs_partition if algo == "partition" else lexbfs_labels
        order = fn(g, tie_break, method=lex_method)
        ok, w = is_peo(g, order)
        return ChordalityVerdict(True, peo=order) if ok else ChordalityVerdict(False, witness=w)
    order, w0 = pipeline.is_chordal(g, _native.TIE_ASCENDING)
    if w0 is None:
        return ChordalityVerdict(True, peo=order)
    return ChordalityVerdict(False, witness=_witness(w0))
