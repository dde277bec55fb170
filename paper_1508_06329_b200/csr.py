"""Sparse graphs in CSR form and their device residency.

The reference stores every graph as a dense bit matrix (graph.py:31-88) and
refuses n above a cap; the N = 10^6 configuration therefore runs its linked
LexBFS and list PEO test on a duck-typed object exposing ``n``, ``m`` and
``adjacency_lists0()``.  ``CSRGraph`` is that object here:
int64 ``indptr`` / int32 ``indices`` (ascending, symmetric), uploaded once to
HBM.  Every entry point of the package accepts it (and any foreign object
with ``adjacency_lists0()`` and no ``_packed``) and routes it to the CSR
kernels (csrc/csr.cu).
"""

from __future__ import annotations

import numpy as np

from . import _native
from .errors import InvalidVertex, SelfLoop


class CSRGraph:
    """Immutable simple undirected graph on 1..n in compressed sparse rows."""

    __slots__ = ("n", "m", "indptr", "indices", "_dev", "_lists0")

    def __init__(self, n: int, indptr: np.ndarray, indices: np.ndarray):
        self.n = int(n)
        self.indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        self.indices = np.ascontiguousarray(indices, dtype=np.int32)
        self.indptr.setflags(write=False)
        self.indices.setflags(write=False)
        self.m = int(self.indptr[-1]) // 2 if self.n else 0
        self._dev = None
        self._lists0 = None

    @classmethod
    def from_edges0(cls, n: int, u: np.ndarray, v: np.ndarray) -> "CSRGraph":
        """0-based endpoints; duplicates collapse, both directions stored."""
        u = np.asarray(u, dtype=np.int64)
        v = np.asarray(v, dtype=np.int64)
        if u.size and ((u < 0).any() or (u >= n).any() or (v < 0).any() or (v >= n).any()):
            raise InvalidVertex(f"edge endpoint outside 0..{n - 1}")
        if (u == v).any():
            raise SelfLoop("self-loop in edge list")
        key = np.unique(np.concatenate([u * n + v, v * n + u]))
        rows, cols = key // n, key % n
        indptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.bincount(rows, minlength=n), out=indptr[1:])
        return cls(n, indptr, cols.astype(np.int32))

    @classmethod
    def from_edge_list(cls, n: int, edges) -> "CSRGraph":
        arr = np.asarray(list(edges) if not isinstance(edges, np.ndarray) else edges, dtype=np.int64)
        if arr.size == 0:
            return cls(n, np.zeros(n + 1, dtype=np.int64), np.zeros(0, dtype=np.int32))
        return cls.from_edges0(n, arr[:, 0] - 1, arr[:, 1] - 1)

    @classmethod
    def from_lists0(cls, lists) -> "CSRGraph":
        n = len(lists)
        deg = np.fromiter((len(x) for x in lists), dtype=np.int64, count=n)
        indptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(deg, out=indptr[1:])
        indices = np.fromiter((y for x in lists for y in x), dtype=np.int32, count=int(indptr[-1]))
        return cls(n, indptr, indices)

    @classmethod
    def from_dense(cls, g) -> "CSRGraph":
        n = int(g.n)
        rows = np.unpackbits(np.asarray(g._packed), axis=1, bitorder="little", count=n).astype(bool)
        indptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(rows.sum(axis=1), out=indptr[1:])
        return cls(n, indptr, (np.flatnonzero(rows.reshape(-1)) % max(n, 1)).astype(np.int32))

    def adjacency_lists0(self) -> list[list[int]]:
        if self._lists0 is None:
            ip, ix = self.indptr, self.indices
            self._lists0 = [ix[ip[v] : ip[v + 1]].tolist() for v in range(self.n)]
        return self._lists0

    def neighbors(self, v: int) -> list[int]:
        if not 1 <= v <= self.n:
            raise InvalidVertex(f"vertex {v} outside 1..{self.n}")
        return (self.indices[self.indptr[v - 1] : self.indptr[v]] + 1).tolist()

    def has_edge(self, u: int, v: int) -> bool:
        if not (1 <= u <= self.n and 1 <= v <= self.n):
            raise InvalidVertex(f"vertex outside 1..{self.n}")
        row = self.indices[self.indptr[u - 1] : self.indptr[u]]
        k = np.searchsorted(row, v - 1)
        return bool(k < row.size and row[k] == v - 1)

    def __repr__(self) -> str:
        return f"CSRGraph(n={self.n}, m={self.m})"


def is_csr(g) -> bool:
    """True for CSR inputs: CSRGraph or a foreign list-only graph (no _packed)."""
    return isinstance(g, CSRGraph) or (not hasattr(g, "_packed") and hasattr(g, "adjacency_lists0"))


def as_csr(g) -> CSRGraph:
    if isinstance(g, CSRGraph):
        return g
    if hasattr(g, "indptr") and hasattr(g, "indices"):
        return CSRGraph(g.n, np.asarray(g.indptr), np.asarray(g.indices))
    return CSRGraph.from_lists0(g.adjacency_lists0())


def device_csr(g):
    """(indptr int64[n+1], indices int32[2m]) device tensors, cached on CSRGraph."""
    torch = _native.require_cuda()
    c = as_csr(g)
    if c._dev is not None and c._dev[0].device.index == torch.cuda.current_device():
        return c._dev
    ip = torch.from_numpy(np.array(c.indptr)).cuda()
    ix = torch.from_numpy(np.array(c.indices) if c.indices.size else np.zeros(1, np.int32)).cuda()
    c._dev = (ip, ix)
    if isinstance(g, CSRGraph):
        g._dev = c._dev
    return c._dev
