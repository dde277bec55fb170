"""The device LexBFS certificate (chordal_lexbfs_certify_dense) behind
lexbfs_labels(debug=True) and parallel_lexbfs(audit=True / debug_labels=True).

The kernel replays the search with forced pivots; its two step indices must
equal the pure-Python label replay of the oracle (oracle.lexbfs_certify, pinned
to the reference's own orders by test_oracle_golden.py) on reference orders,
corrupted orders and random permutations, in both the one-warp and the
multi-warp forms of the engine.
"""

import numpy as np
import pytest

import oracle
import paper_1508_06329_b200 as P
from paper_1508_06329_b200 import pipeline
from paper_1508_06329_b200.csr import CSRGraph
from paper_1508_06329_b200.errors import GraphTooLarge
from paper_1508_06329_b200.generate import gen_chordal_random, gen_dense_random
from paper_1508_06329_b200.parallel import Arbitration

pytestmark = pytest.mark.gpu


def G(packed, n):
    return P.Graph._from_packed(n, np.array(packed, dtype=np.uint8, copy=True))


def cert(g, order0):
    return pipeline.certify_lexbfs(g, P.VertexOrdering.from_zero_based(list(order0)))


def test_certificate_matches_oracle_on_reference_orders(small_corpus):
    c = small_corpus
    for i in range(0, len(c), 2):
        n = int(c.ns[i])
        g = G(c.packed(i), n)
        for key in ("lex", "par_desc", "par_seeded", "seeded_array", "perm"):
            o = c.vec(key, i).tolist()
            assert cert(g, o) == oracle.lexbfs_certify(c.packed(i), n, o), (i, key)


@pytest.mark.parametrize("n,k", [(300, 6), (1500, 8), (3000, 40)])
def test_certificate_on_corrupted_orders(n, k):
    """A LexBFS order with two positions swapped: the kernel names the same
    first bad step as the label replay (sparse graphs: one-warp engine up to
    n = 16384; k = 40 at n = 3000 is still sparse)."""
    g = gen_chordal_random(n, k, 11)
    lex = P.lexbfs_partition(g).order0.tolist()
    assert cert(g, lex) == (-1, -1)
    rng = np.random.default_rng(n)
    for _ in range(4 if n <= 300 else 2):
        a, b = sorted(rng.choice(n, 2, replace=False).tolist())
        o = list(lex)
        o[a], o[b] = o[b], o[a]
        want = oracle.lexbfs_certify(g._packed, n, o) if n <= 1500 else None
        got = cert(g, o)
        if want is not None:
            assert got == want, (a, b)
        assert got[0] == -1 or got[0] >= a


def test_certificate_dense_multiwarp():
    g = gen_dense_random(2500, 0.5, 3)
    lex = P.lexbfs_partition(g).order0.tolist()
    assert cert(g, lex) == (-1, -1)
    o = list(lex)
    o[5], o[2000] = o[2000], o[5]
    bad, off = cert(g, o)
    assert off == 5 and (bad == -1 or bad >= 5)


def test_debug_and_audit_entry_points():
    g = gen_chordal_random(2000, 8, 4)
    base = P.lexbfs_partition(g).order0.tolist()
    assert P.lexbfs_labels(g, debug=True).order0.tolist() == base
    assert P.parallel_lexbfs(g, Arbitration.fixed_priority(), audit=True).order0.tolist() == base
    for arb in (Arbitration.fixed_priority("descending"), Arbitration.seeded(5)):
        o = P.parallel_lexbfs(g, arb, debug_labels=True)
        assert cert(g, o.order0.tolist())[0] == -1
    small = gen_chordal_random(200, 5, 2)
    o = P.lexbfs_labels(small, P.seeded(3), debug=True)  # linked seeded labels on the slot engine
    assert cert(small, o.order0.tolist())[0] == -1
    csr = CSRGraph.from_dense(g)
    assert P.lexbfs_labels(csr, debug=True).order0.tolist() == base
    assert cert(csr, base) == (-1, -1)


def test_certificate_size_limit():
    from paper_1508_06329_b200.generate import chordal_random_edges

    n = 40000
    u, v = chordal_random_edges(n, 3, 0)
    g = CSRGraph.from_edges0(n, u, v)
    with pytest.raises(GraphTooLarge):
        P.lexbfs_labels(g, debug=True)
