"""Two-phase parallel PEO test and the parallel chordality pipeline (paper §6.2).

``parallel_peo_test`` / ``parallel_is_chordal`` keep the reference signatures
(parallel/peo.py:68-114).  The paper's preparationLNandP and testing kernels
 are one vertex-parallel CUDA kernel (csrc/peo_dense.cu);
the pipeline runs LexBFS and the test back to back on one stream, and a
failing run carries the same deterministic witness the sequential scan
extracts from the parallel ordering (parallel/peo.py:113).
"""

from __future__ import annotations

from .. import pipeline
from ..errors import InvalidOrdering
from ..graph import as_ordering
from ..peo import ChordalityVerdict, WitnessTriple
from .engine import Arbitration
from .lexbfs import _check_backend


def parallel_peo_test(g, ordering, *, backend: str = "auto", workers: int = 1) -> bool:
    """Elimination-order check; the verdict carries no witness (parallel/peo.py:68-95)."""
    o = as_ordering(ordering)
    if o.n != g.n:
        raise InvalidOrdering(f"ordering covers {o.n} vertices, graph has {g.n}")
    _check_backend(backend, False, False, False)
    if g.n == 0:
        return True
    return pipeline.peo_witness(g, o) is None


def parallel_is_chordal(g, arb: Arbitration, *, backend: str = "auto",
                        workers: int = 1) -> ChordalityVerdict:
    """Parallel LexBFS followed by the parallel PEO test (parallel/peo.py:98-114)."""
    _check_backend(backend, False, False, False)
    order, w0 = pipeline.is_chordal(g, arb.tie_rule, arb.seed or 0)
    if w0 is None:
        return ChordalityVerdict(True, peo=order)
    return ChordalityVerdict(False, witness=WitnessTriple(w0[0] + 1, w0[1] + 1, w0[2] + 1))
