"""Barrier-synchronised LexBFS (paper §6.1) as one persistent CUDA kernel.

``parallel_lexbfs`` keeps the reference signature (parallel/lexbfs.py:234-243).
The paper launches four kernels per step and the reference
replays them as four barrier phases over a linked set list
(parallel/lexbfs.py:37-231); here one CTA runs every step between
__syncthreads barriers (csrc/lexbfs_dense.cu) and the ``current`` election of
kernel 4 is the kernel's tie rule:
  fixed ascending  -> smallest id of the max-label set (= LOWEST_INDEX),
  fixed descending -> largest id,
  seeded(s)        -> argmax (splitmix64(prefix_i ^ w), w), prefix_i =
                      mix64(s, 4(i-1)+3, mix64(crc32("current"), 0)).
Every rule starts at vertex 1 (parallel/lexbfs.py:173).  The other racy writes
of kernels 2-4 (set splices, counters) never change the order.
"""

from __future__ import annotations

from .. import pipeline
from ..graph import VertexOrdering
from .engine import Arbitration

_VECTOR_MIN_N = 128  # the reference's backend threshold (parallel/lexbfs.py:30)


def _check_backend(backend: str, audit: bool, debug_labels: bool, adj_reuse: bool) -> None:
    if backend not in ("auto", "tasks", "vector"):
        raise ValueError(f"unknown backend {backend!r}")
    if backend == "vector" and (audit or debug_labels or adj_reuse):
        raise ValueError("audit, debug_labels and adj_reuse need the tasks backend")


def parallel_lexbfs(g, arb: Arbitration, *, backend: str = "auto", workers: int = 1,
                    debug_labels: bool = False, audit: bool = False,
                    adj_reuse: bool = False) -> VertexOrdering:
    """LexBFS via the paper's barrier-phase algorithm; starts at vertex 1.

    ``backend``/``workers``/``adj_reuse`` select CPU execution strategies in
    the reference; they are validated the same way and all run the same CUDA
    kernel (its output is independent of them in the reference too,
    test_parallel_lexbfs.py:98-137, 152-184).  ``audit`` / ``debug_labels``
    (the reference checks its set-list invariants after every phase,
    parallel/lexbfs.py:82-129) replay the finished order on the device with its
    pivots forced and assert that every elected ``current`` carries the largest
    label -- under fixed ascending priority also that it is the smallest id of
    its set (search._certified).
    """
    _check_backend(backend, audit, debug_labels, adj_reuse)
    o = pipeline.lexbfs(g, arb.tie_rule, arb.seed or 0)
    if audit or debug_labels:
        from ..search import _certified

        exact = arb.mode == "fixed" and arb.direction == "ascending"
        _certified(g, o, exact, "parallel_lexbfs(audit=True)" if audit else "parallel_lexbfs(debug_labels=True)")
    return o
