"""Left neighbourhoods, parents and ScanStats on the GPU, and the seeded tie
rules at sizes where the reference takes its array / vector paths.

Checked against fixtures frozen from the reference (left_scan.npz,
seeded_large.npz; tests/golden/make_left_golden.py) and the oracle.
"""

import numpy as np
import pytest
import torch

import oracle
import paper_1508_06329_b200 as P
from conftest import load_npz
from paper_1508_06329_b200 import ops
from paper_1508_06329_b200.csr import CSRGraph, device_csr
from paper_1508_06329_b200.device import device_rows
from paper_1508_06329_b200.generate import chordal_random_edges, gen_chordal_random, gen_dense_random
from paper_1508_06329_b200.parallel import Arbitration

pytestmark = pytest.mark.gpu


def G(packed, n):
    return P.Graph._from_packed(n, np.array(packed, dtype=np.uint8, copy=True))


def ln_sets(packed, n, order0):
    """LN(v) by definition (graph.py:284-302), 1-based sets."""
    pos = np.empty(n, dtype=np.int64)
    pos[order0] = np.arange(n)
    rows = np.unpackbits(np.asarray(packed), axis=1, bitorder="little", count=n).astype(bool)
    return [set((np.flatnonzero(rows[v] & (pos < pos[v])) + 1).tolist()) for v in range(n)]


def test_left_neighborhoods_match_reference(left_corpus):
    c = left_corpus
    for i in range(len(c)):
        n = int(c.ns[i])
        g = G(c.packed(i), n)
        o = P.VertexOrdering.from_zero_based(c.vec("order", i))
        ln = P.left_neighborhoods(g, o)
        par = c.vec("parent", i)
        assert [ln.parent(v) for v in range(1, n + 1)] == [None if p < 0 else int(p) + 1 for p in par], i
        assert [len(ln.ln(v)) for v in range(1, n + 1)] == c.vec("ln_size", i).tolist(), i
        if i % 25 == 0:
            assert [ln.ln(v) for v in range(1, n + 1)] == ln_sets(c.packed(i), n, c.vec("order", i)), i
        assert ln.ordering == o


def test_scan_stats_match_reference_dense_and_csr(left_corpus):
    """ScanStats of is_peo(g, o, stats=...) equal the reference's list scan counts
    (600 frozen cases), for packed-row graphs and for the same graphs in CSR."""
    c = left_corpus
    z = c.z
    for i in range(len(c)):
        n = int(c.ns[i])
        g = G(c.packed(i), n)
        o = P.VertexOrdering.from_zero_based(c.vec("order", i))
        want_w = None if z["witness"][i][0] < 0 else P.WitnessTriple(*(int(x) + 1 for x in z["witness"][i]))
        forms = (g, CSRGraph.from_dense(g)) if i % 3 == 0 else (g,)
        for gg in forms:
            st = P.ScanStats()
            ok, w = P.is_peo(gg, o, stats=st)
            assert ok == bool(z["ok"][i]) and w == want_w, (i, type(gg).__name__)
            assert (st.reads, st.budget) == (int(z["reads"][i]), int(z["budget"][i])), (i, type(gg).__name__)


def test_left_parents_equal_lexbfs_parents_and_oracle():
    """The device parent search (csrc/left.cu) against the oracle's scan 1 on
    larger graphs, and against the parents LexBFS records during the search
    (every engine: CTA engine n <= 32768, slot engine on CSR and n > 32768)."""
    cases = [
        ("chordal2000", gen_chordal_random(2000, 8, 1)),
        ("dense3000", gen_dense_random(3000, 0.2, 2)),
        ("chordal20000", gen_chordal_random(20000, 6, 3, cap=20000)),
    ]
    rng = np.random.default_rng(7)
    for name, g in cases:
        n = g.n
        ip, ix = oracle.csr_from_packed(g._packed, n)
        rows = device_rows(g)
        order, pos, par = ops.lexbfs(rows, want_parent=True)
        o0 = order.cpu().numpy()
        perm = rng.permutation(n).astype(np.int32)
        for oo in (o0, perm):
            _, _, want_par, want_ln, _ = oracle.peo_lists_stats(ip, ix, n, oo)
            ln = P.left_neighborhoods(g, P.VertexOrdering.from_zero_based(oo))
            got = np.array([-1 if ln.parent(v) is None else ln.parent(v) - 1 for v in range(1, n + 1)])
            assert np.array_equal(got, want_par), name
            od = torch.as_tensor(oo.astype(np.int32)).cuda()
            gp, gl = ops.left_csr(*device_csr(CSRGraph(n, ip, ix)), n, od, ops.positions(od))
            assert np.array_equal(gp[:n].cpu().numpy(), want_par) and np.array_equal(gl[:n].cpu().numpy(), want_ln)
        _, _, want_par, _, _ = oracle.peo_lists_stats(ip, ix, n, o0)
        lp = par.cpu().numpy()
        known = lp != -2  # -2: placed by the early exit, the PEO check searches it
        assert np.array_equal(lp[known], want_par[known]), name
        # the slot engine's parents (CSR input)
        c = CSRGraph(n, ip, ix)
        dip, dix = device_csr(c)
        o5, _, p5 = ops.lexbfs_csr(dip, dix, n)
        assert np.array_equal(o5.cpu().numpy(), o0), name
        sp = p5.cpu().numpy()
        known = sp != -2
        assert np.array_equal(sp[known], want_par[known]), name


def test_left_csr_large_parents_and_stats():
    """CSR n = 200000 (config-5 shape, scaled): parents / |LN| and ScanStats against
    the oracle's literal list scan, for the LexBFS order and a chord-breaking swap."""
    n = 200_000
    u, v = chordal_random_edges(n, 8, 5)
    g = CSRGraph.from_edges0(n, u, v)
    o = P.lexbfs_partition(g)
    for order0 in (o.order0, np.concatenate([o.order0[:50][::-1], o.order0[50:]])):
        ok, w, par, lnsz, reads = oracle.peo_lists_stats(g.indptr, g.indices, n, order0)
        oo = P.VertexOrdering.from_zero_based(order0)
        st = P.ScanStats()
        got_ok, got_w = P.is_peo(g, oo, stats=st)
        assert got_ok == ok
        assert (None if got_w is None else (got_w.v - 1, got_w.p - 1, got_w.z - 1)) == w
        assert st.reads == reads and st.budget == 8 * g.m


def test_left_neighborhoods_errors_and_empty():
    g = P.Graph.from_edge_list(3, [(1, 2)])
    with pytest.raises(P.InvalidOrdering):
        P.left_neighborhoods(g, P.VertexOrdering([1, 2]))
    e = P.left_neighborhoods(P.Graph.from_edge_list(0, []), P.VertexOrdering(()))
    assert e.ordering.n == 0
    ln = P.left_neighborhoods(g, P.VertexOrdering([2, 3, 1]))
    assert ln.ln(1) == {2} and ln.parent(1) == 2 and ln.parent(2) is None and ln.ln(3) == set()
    with pytest.raises(P.InvalidVertex):
        ln.ln(4)


SEEDED = load_npz("seeded_large.npz")


@pytest.mark.parametrize("name,mk,seed", [
    ("array_chordal2048_s7", lambda: gen_chordal_random(2048, 8, 3), 7),
    ("array_dense2048_s5", lambda: gen_dense_random(2048, 0.3, 4), 5),
    ("array_chordal8192_s11", lambda: gen_chordal_random(8192, 8, 0), 11),
])
def test_seeded_array_method_large(name, mk, seed):
    """lexbfs_partition / lexbfs_labels (seeded, method="array" = the auto path at
    n >= 1024, search.py:535-541): the device relabel + ascending kernel against
    the reference's frozen order and the oracle's lexbfs_array with the same
    Philox initial arrangement."""
    g = mk()
    want = SEEDED[name].astype(np.int64)
    got = P.lexbfs_partition(g, P.seeded(seed)).order0
    assert np.array_equal(got, want)
    initial = P.seeded(seed).generator("lexbfs-partition").permutation(g.n)
    assert np.array_equal(oracle.lexbfs_array(g._packed, g.n, initial), want)
    lab = P.lexbfs_labels(g, P.seeded(seed), method="array").order0
    ini_l = P.seeded(seed).generator("lexbfs-labels").permutation(g.n)
    assert np.array_equal(lab, oracle.lexbfs_array(g._packed, g.n, ini_l))


def test_seeded_arbitration_on_global_slot_engine():
    """parallel_lexbfs(Arbitration.seeded(3)) on a dense-stored graph of 40000
    vertices: above the shared-memory engines' 32768, so it runs on the
    global-memory slot engine.  Against the reference's frozen order (24.9 s in
    the reference) and the oracle's arbitrated LexBFS."""
    g = gen_chordal_random(40000, 4, 2, cap=40000)
    want = SEEDED["parseeded_chordal40000_k4_s3"].astype(np.int64)
    got = P.parallel_lexbfs(g, Arbitration.seeded(3)).order0
    assert np.array_equal(got, want)
    assert np.array_equal(oracle.lexbfs_arbitrated(g._packed, g.n, oracle.ARB_SEEDED, 3), want)
    v = P.parallel_is_chordal(g, Arbitration.seeded(3))
    assert v.chordal and np.array_equal(v.peo.order0, want)
