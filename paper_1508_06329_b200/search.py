"""LexBFS orderings -- the reference's ``chordalkit.search`` entry points on the GPU.

``lexbfs_labels`` (search.py:262-310) and ``lexbfs_partition``
(search.py:500-532) keep their signatures and return types; both run the
persistent single-CTA kernel of ``csrc/lexbfs_seg.cu`` (n <= 32768; larger
graphs the CSR slot engine).  Under the default
``LOWEST_INDEX`` tie-break every reference method ("linked", "array",
"auto") yields the same order (the reference's own equality tests,
test_search.py:98-112), and so does this one.

Seeded tie-breaks are method-dependent in the reference:
``method="array"`` (and "auto" for n >= 1024) breaks ties by a Philox
permutation of the vertices (search.py:535-541); that is replayed here by
relabelling the graph on the device with the same permutation and running the
ascending kernel.  The linked seeded variants (n < 1024 under "auto") run
the CSR slot engine with the reference's random choices replayed from the
same Philox streams: ``lexbfs_partition`` shuffles the initial class
(Generator.shuffle) and keeps split-off classes in adjacency order,
``lexbfs_labels`` draws the pivot's index in the max-label class
(Generator.integers) at every step.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native, ops, pipeline
from .csr import is_csr
from .device import device_rows
from .graph import VertexOrdering

_ARRAY_MIN_N = 1024  # the reference's auto-dispatch threshold (search.py:29)


@dataclass(frozen=True)
class TieBreak:
    """How to pick among equally eligible vertices (search.py:32-41)."""

    seed: int | None = None

    def generator(self, label: str):
        if self.seed is None:
            return None
        from .generate import stream

        return stream(self.seed, label)


LOWEST_INDEX = TieBreak()


def seeded(seed: int) -> TieBreak:
    return TieBreak(int(seed))


@dataclass(frozen=True)
class LexLabel:
    """A lexicographic label: digits appended over time, strictly falling (search.py:51-69)."""

    digits: tuple[int, ...] = ()

    def __post_init__(self):
        d = self.digits
        if any(b >= a for a, b in zip(d, d[1:])):
            raise ValueError(f"label digits must strictly descend: {d}")

    def extended(self, digit: int) -> "LexLabel":
        return LexLabel(self.digits + (digit,))

    def __lt__(self, other: "LexLabel") -> bool:
        return self.digits < other.digits

    def __le__(self, other: "LexLabel") -> bool:
        return self.digits <= other.digits


def _run_lexbfs(g, tie_break: TieBreak, label: str, method: str) -> VertexOrdering:
    n = int(g.n)
    if tie_break.seed is None:
        return pipeline.lexbfs(g, _native.TIE_ASCENDING)
    if method == "linked":
        # per-split / per-step random choices of the linked structures
        # (search.py:285-290 labels, 515-518 partition), replayed by the slot engine
        rule = _native.TIE_SEEDED_LABELS if label == "lexbfs-labels" else _native.TIE_SEEDED_PARTITION
        return pipeline.lexbfs_linked_seeded(g, rule, int(tie_break.seed))
    if is_csr(g):
        raise NotImplementedError("the seeded array method needs the dense rows (it relabels the matrix)")
    if n == 0:
        return VertexOrdering(())
    initial = np.asarray(tie_break.generator(label).permutation(n), dtype=np.int64)
    perm = ops.permute(device_rows(g), initial)
    order_r, _ = ops.lexbfs(perm, _native.TIE_ASCENDING)
    return VertexOrdering._trusted(initial[order_r.cpu().numpy()])


def _certified(g, o: VertexOrdering, exact_lowest: bool, what: str) -> VertexOrdering:
    """Device check of the LexBFS label invariant on the order just produced
    (pipeline.certify_lexbfs): every pivot has the largest label among the
    unvisited vertices -- what the reference's debug chain check and audit
    lemmas assert -- and, under LOWEST_INDEX, every pivot is the smallest id of
    its label class."""
    bad, off_rule = pipeline.certify_lexbfs(g, o)
    if bad >= 0:
        raise AssertionError(f"{what}: the pivot of step {bad + 1} does not carry the largest label")
    if exact_lowest and off_rule >= 0:
        raise AssertionError(f"{what}: step {off_rule + 1} is not the LOWEST_INDEX choice")
    return o


def lexbfs_labels(g, tie_break: TieBreak = LOWEST_INDEX, *, debug: bool = False,
                  method: str = "auto") -> VertexOrdering:
    """Lexicographic BFS (label-class formulation, search.py:262-310) on the GPU.

    ``debug=True`` (search.py:270-271: labels materialised, the chain checked
    after every step) replays the finished order on the device with its pivots
    forced and asserts the same invariant at every step (``_certified``).
    """
    if method not in ("auto", "array", "linked"):
        raise ValueError(f"unknown method {method!r}")
    if method == "auto":
        method = "array" if g.n >= _ARRAY_MIN_N and not debug else "linked"
    o = _run_lexbfs(g, tie_break, "lexbfs-labels", method)
    if debug:
        _certified(g, o, tie_break.seed is None, "lexbfs_labels(debug=True)")
    return o


def lexbfs_partition(g, tie_break: TieBreak = LOWEST_INDEX, *, method: str = "auto",
                     _watch=None) -> VertexOrdering:
    """Lexicographic BFS (partition refinement, search.py:500-532) on the GPU."""
    if method not in ("auto", "array", "linked"):
        raise ValueError(f"unknown method {method!r}")
    if _watch is not None:
        # a per-step Python callback on the reference's CPU PartitionList object;
        # the persistent kernel has no such object to hand out between steps
        raise NotImplementedError("_watch observes the CPU PartitionList; the GPU search has none "
                                  "(lexbfs_labels(debug=True) checks the label invariant on the device)")
    if method == "auto":
        method = "array" if g.n >= _ARRAY_MIN_N else "linked"
    return _run_lexbfs(g, tie_break, "lexbfs-partition", method)


def bfs_order(g, tie_break: TieBreak = LOWEST_INDEX) -> VertexOrdering:
    """A breadth-first visit order (FIFO queue, component restarts; search.py:79-110) on the GPU."""
    return pipeline.bfs_order(g, tie_break.seed is not None, int(tie_break.seed or 0))


def mcs_order(g, tie_break: TieBreak = LOWEST_INDEX) -> VertexOrdering:
    """Maximum cardinality search (search.py:113-145) on the GPU: repeatedly visit an
    unvisited vertex with the most visited neighbours."""
    return pipeline.mcs_order(g, tie_break.seed is not None, int(tie_break.seed or 0))
