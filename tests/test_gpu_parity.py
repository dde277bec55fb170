"""Parity of the CUDA path (through libchordal_b200.so) with the reference.

Checked against (a) fixtures frozen from the reference itself
(tests/golden/) and (b) the CPU oracle (oracle/, itself pinned to those
fixtures by test_oracle_golden.py) on seeded inputs.  Integer / index work:
everything must be bit-exact -- identical orders, verdicts and witnesses.
"""

import ctypes
import hashlib
import os

import numpy as np
import pytest

import oracle
import paper_1508_06329_b200 as P
from conftest import GOLDEN, exhaustive_graph_packed, load_json, load_npz, named_packed
from paper_1508_06329_b200 import _native
from paper_1508_06329_b200.generate import (
    gen_chordal_random,
    gen_dense_random,
    gen_dense_random_device,
    packed_sha256,
    remove_first_chord,
)
from paper_1508_06329_b200.parallel import Arbitration

pytestmark = pytest.mark.gpu

ASC = Arbitration.fixed_priority()
DESC = Arbitration.fixed_priority("descending")
NAMED = load_json("named.json")
CONFIGS = load_json("configs.json") if os.path.exists(os.path.join(GOLDEN, "configs.json")) else {}


def G(packed, n):
    return P.Graph._from_packed(n, np.array(packed, dtype=np.uint8, copy=True))


def o0(ordering):
    return ordering.order0.tolist()


def w0(w):
    return None if w is None else [w.v - 1, w.p - 1, w.z - 1]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---------------------------------------------------------------- goldens ----


@pytest.mark.parametrize("rec", NAMED["graphs"], ids=[r["name"] for r in NAMED["graphs"]])
def test_named_goldens(rec):
    g = G(named_packed(rec), rec["n"])
    assert o0(P.lexbfs_partition(g)) == rec["lexbfs_partition"]
    assert o0(P.lexbfs_labels(g)) == rec["lexbfs_labels"]
    assert o0(P.parallel_lexbfs(g, ASC)) == rec["par_asc"]
    assert o0(P.parallel_lexbfs(g, DESC)) == rec["par_desc"]
    for s, o in rec["par_seeded"].items():
        assert o0(P.parallel_lexbfs(g, Arbitration.seeded(int(s)))) == o
    v = P.is_chordal(g)
    assert v.chordal == rec["chordal"] and w0(v.witness) == rec["witness"]
    if v.chordal:
        assert o0(v.peo) == rec["lexbfs_partition"]
    pv = P.parallel_is_chordal(g, Arbitration.seeded(6))
    assert pv.chordal == rec["par_seeded6_chordal"] and w0(pv.witness) == rec["par_seeded6_witness"]


def test_frozen_values_of_the_reference_suite():
    graphs = {r["name"]: G(named_packed(r), r["n"]) for r in NAMED["graphs"]}
    c4 = graphs["c4"]
    assert list(P.lexbfs_partition(c4)) == [1, 2, 4, 3]            # test_search.py:34-39
    assert list(P.parallel_lexbfs(c4, DESC)) == [1, 4, 2, 3]        # test_parallel_lexbfs.py:54-57
    ok, w = P.is_peo(c4, P.VertexOrdering([1, 2, 4, 3]))           # test_peo.py:39-43
    assert not ok and (w.v, w.p, w.z) == (3, 4, 2) and w.verify(c4, P.VertexOrdering([1, 2, 4, 3]))
    assert list(P.lexbfs_partition(graphs["p3_relabeled"])) == [1, 3, 2]
    assert list(P.lexbfs_partition(graphs["disconnected6"])) == [1, 3, 2, 5, 6, 4]
    assert list(P.is_chordal(graphs["clique4"]).peo) == [1, 2, 3, 4]
    assert P.parallel_peo_test(graphs["star5"], P.VertexOrdering([2, 3, 4, 5, 1])) is False
    assert P.parallel_peo_test(graphs["star5"], P.VertexOrdering([1, 2, 3, 4, 5])) is True


def test_frozen_peo_cases():
    graphs = {r["name"]: r for r in NAMED["graphs"]}
    for case in NAMED["peo_cases"]:
        rec = graphs[case["graph"]]
        g = G(named_packed(rec), rec["n"])
        ok, w = P.is_peo(g, P.VertexOrdering.from_zero_based(case["order"]))
        assert ok == case["ok"] and w0(w) == case["witness"]


def test_random_small_goldens(small_corpus):
    c = small_corpus
    for i in range(len(c)):
        n = int(c.ns[i])
        g = G(c.packed(i), n)
        assert o0(P.lexbfs_partition(g)) == c.vec("lex", i).tolist(), i
        assert o0(P.parallel_lexbfs(g, DESC)) == c.vec("par_desc", i).tolist(), i
        assert o0(P.parallel_lexbfs(g, Arbitration.seeded(i))) == c.vec("par_seeded", i).tolist(), i
        assert o0(P.lexbfs_partition(g, P.seeded(i), method="array")) == c.vec("seeded_array", i).tolist(), i
        ok, w = P.is_peo(g, P.VertexOrdering.from_zero_based(c.vec("perm", i)))
        assert ok == bool(c.z["perm_ok"][i])
        assert (w0(w) or [-1, -1, -1]) == c.z["perm_witness"][i].tolist(), i
        v = P.is_chordal(g)
        assert (w0(v.witness) or [-1, -1, -1]) == c.z["chordal_witness"][i].tolist(), i


def test_exhaustive5_single_and_batch():
    z = load_npz("exhaustive5.npz")
    for n in range(1, 6):
        idx = np.flatnonzero(z["n"] == n)
        graphs = [G(exhaustive_graph_packed(n, int(z["mask"][k])), n) for k in idx]
        bv = P.is_chordal_batch(graphs)
        for j, k in enumerate(idx):
            assert bv.orders0[j].tolist() == z["order"][k][:n].tolist()
            assert bool(bv.chordal[j]) == bool(z["chordal"][k])
            assert bv.witness0[j].tolist() == z["witness"][k].tolist()
        for j in range(0, len(idx), 7):
            v = P.is_chordal(graphs[j])
            assert (w0(v.witness) or [-1, -1, -1]) == z["witness"][idx[j]].tolist()


# ------------------------------------------------------- oracle, larger n ----


def _random_cases():
    out = []
    for n, kind, seed in [(100, "dense", 1), (257, "chordal", 2), (500, "dense", 3), (1000, "chordal", 4),
                          (1000, "sparse", 5), (2048, "chordal", 6), (3000, "dense", 7), (5000, "chordal", 8),
                          (8191, "sparse", 9), (12000, "chordal", 10), (16000, "dense", 11), (20000, "sparse", 12)]:
        if kind == "dense":
            g = gen_dense_random(n, 0.5, seed)
        elif kind == "sparse":
            g = gen_dense_random(n, 4.0 / n, seed)
        else:
            g = gen_chordal_random(n, 6, seed)
        out.append((f"{kind}{n}", g))
        if kind == "chordal":
            h, _ = remove_first_chord(g)
            out.append((f"{kind}{n}-chord", h))
    return out


@pytest.mark.parametrize("name,g", _random_cases(), ids=[c[0] for c in _random_cases()])
def test_against_oracle(name, g):
    n = g.n
    ok, order, w = oracle.is_chordal(g._packed, n)
    v = P.is_chordal(g)
    assert v.chordal == ok
    assert o0(P.lexbfs_partition(g)) == order.tolist()
    assert w0(v.witness) == (None if w is None else list(w))
    # arbitrary orderings exercise the parent search's full-row fallback
    rng = np.random.default_rng(n)
    perm = rng.permutation(n)
    ok2, w2 = oracle.is_peo(g._packed, n, perm)
    okg, wg = P.is_peo(g, P.VertexOrdering.from_zero_based(perm))
    assert okg == ok2 and w0(wg) == (None if w2 is None else list(w2))
    assert P.parallel_peo_test(g, P.VertexOrdering.from_zero_based(perm)) is ok2
    for arb, mode, seed in ((DESC, oracle.ARB_DESCENDING, 0), (Arbitration.seeded(n), oracle.ARB_SEEDED, n)):
        assert o0(P.parallel_lexbfs(g, arb)) == oracle.lexbfs_arbitrated(g._packed, n, mode, seed).tolist()


# ---------------------------------------------------------------- configs ----


@pytest.mark.skipif("1" not in CONFIGS, reason="configs.json not generated")
def test_config1():
    orders = load_npz("configs_orders.npz")
    g = gen_chordal_random(1000, 8, 0)
    h, _ = remove_first_chord(g)
    for graph, key, okey in ((g, "chordal", "c1_chordal"), (h, "nonchordal", "c1_nonchordal")):
        exp = CONFIGS["1"][key]
        v = P.is_chordal(graph)
        assert v.chordal == exp["chordal"] and w0(v.witness) == exp["witness"]
        assert o0(P.lexbfs_partition(graph)) == orders[okey].astype(int).tolist()
    assert w0(P.is_chordal(h).witness) == [1, 873, 2]  # (v=2, p=874, z=3), SURVEY §8d


@pytest.mark.skipif("2" not in CONFIGS, reason="configs.json not generated")
def test_config2():
    orders = load_npz("configs_orders.npz")
    d = P.Graph._from_packed(8192, gen_dense_random_device(8192, 0.5, 0)[0, :, :1024].cpu().numpy())
    assert packed_sha256(d._packed) == CONFIGS["2"]["dense"]["packed_sha256"]
    c = gen_chordal_random(8192, 8, 0)
    assert packed_sha256(c._packed) == CONFIGS["2"]["chordal"]["packed_sha256"]
    for graph, key, okey in ((d, "dense", "c2_dense"), (c, "chordal", "c2_chordal")):
        exp = CONFIGS["2"][key]
        v = P.is_chordal(graph)
        assert v.chordal == exp["chordal"] and w0(v.witness) == exp["witness"]
        assert o0(P.lexbfs_partition(graph)) == orders[okey].astype(int).tolist()


@pytest.mark.skipif("3" not in CONFIGS, reason="configs.json not generated")
def test_config3_dense_stressor():
    exp = CONFIGS["3"]["dense"]
    adj = gen_dense_random_device(32768, 0.5, 0)
    d = P.Graph._from_packed(32768, adj[0].cpu().numpy())
    assert packed_sha256(d._packed) == exp["packed_sha256"]
    v = P.is_chordal(d)
    assert v.chordal == exp["chordal"] and w0(v.witness) == exp["witness"]
    assert sha(P.lexbfs_partition(d).order0.astype(np.int32)) == exp["order_sha256"]


@pytest.mark.slow
@pytest.mark.skipif("3" not in CONFIGS, reason="configs.json not generated")
def test_config3_chordal_pair():
    g = gen_chordal_random(32768, 1024, 0, cap=32768)
    exp = CONFIGS["3"]["chordal"]
    assert packed_sha256(g._packed) == exp["packed_sha256"]
    v = P.is_chordal(g)
    assert v.chordal and sha(v.peo.order0.astype(np.int32)) == exp["order_sha256"]
    h, e = remove_first_chord(g)
    expn = CONFIGS["3"]["nonchordal"]
    assert list(e) == expn["removed_edge"]
    vn = P.is_chordal(h)
    assert not vn.chordal and w0(vn.witness) == expn["witness"]  # (v=2, p=3600, z=3)
    assert sha(P.lexbfs_partition(h).order0.astype(np.int32)) == expn["order_sha256"]


@pytest.mark.skipif("4" not in CONFIGS, reason="configs.json not generated")
def test_config4_sample_batch():
    sample = CONFIGS["4"]["sample"]
    graphs = [gen_dense_random(512, 0.5, r["seed"]) if r["seed"] % 2 == 0 else gen_chordal_random(512, 8, r["seed"])
              for r in sample]
    bv = P.is_chordal_batch(graphs)
    for b, r in enumerate(sample):
        assert sha(bv.orders0[b].astype(np.int32)) == r["order_sha256"]
        assert bool(bv.chordal[b]) == r["chordal"]
        assert (None if bv.chordal[b] else bv.witness0[b].tolist()) == r["witness"]


def test_batch_against_oracle_mixed_sizes():
    for n in (17, 64, 100, 512, 700, 1024):
        gs = [gen_dense_random(n, [0.05, 0.5, 0.9][s % 3], s) if s % 2 == 0 else gen_chordal_random(n, 5, s)
              for s in range(24)]
        gs += [remove_first_chord(gen_chordal_random(n, 5, 100 + s))[0] for s in range(8)]
        bv = P.is_chordal_batch(gs)
        verdict, orders, wit = oracle.is_chordal_batch(np.stack([g._packed for g in gs]), n)
        assert (bv.chordal == verdict).all()
        assert (bv.orders0 == orders).all()
        assert (bv.witness0 == wit).all()


# ------------------------------------------------------- inputs and e2e ----


def test_device_dense_generator_bit_exact():
    for n, p, seeds in ((512, 0.5, range(0, 8, 2)), (1000, 0.3, range(3, 5)), (33, 0.7, range(1)), (2, 1.0, range(1))):
        adj = gen_dense_random_device(n, p, seeds).cpu().numpy()
        w = (n + 7) // 8
        for b, s in enumerate(seeds):
            ref = gen_dense_random(n, p, s)._packed
            assert (adj[b, :, :w] == ref).all(), (n, s)
            assert not adj[b, :, w:].any()


def test_device_chordal_generator_bit_exact():
    from paper_1508_06329_b200.generate import gen_chordal_random_device

    for n, k, seeds in ((512, 8, range(1, 17, 2)), (300, 30, range(2, 4)), (64, 0, range(1)), (1, 0, range(1)),
                        (1000, 8, range(0, 1)), (50, 49, range(3, 4))):
        adj = gen_chordal_random_device(n, k, seeds).cpu().numpy()
        w = (n + 7) // 8
        for b, s in enumerate(seeds):
            ref = gen_chordal_random(n, k, s)._packed
            assert (adj[b, :, :w] == ref).all(), (n, k, s)
            assert not adj[b, :, w:].any()


def test_edges_to_dense():
    from paper_1508_06329_b200 import ops
    from paper_1508_06329_b200.generate import chordal_random_edges

    u, v = chordal_random_edges(2000, 12, 4)
    rows = ops.edges_to_dense(u, v, 2000, 256).cpu().numpy()
    assert (rows[:, :250] == gen_chordal_random(2000, 12, 4)._packed).all() and not rows[:, 250:].any()


def test_host_buffer_batch_entry_point():
    import torch

    gs = [gen_dense_random(512, 0.5, s) if s % 2 == 0 else gen_chordal_random(512, 8, s) for s in range(40)]
    host = np.zeros((40, 512, 64), dtype=np.uint8)
    for b, g in enumerate(gs):
        host[b] = g._packed
    orders = np.empty((40, 512), dtype=np.int32)
    wit = np.empty((40, 3), dtype=np.int32)
    rc = _native.lib.chordal_is_chordal_batch_host(host.ctypes.data, 40, 512, 64, orders.ctypes.data,
                                                   wit.ctypes.data, 7)  # ragged final chunk
    assert rc == 0
    verdict, o, w = oracle.is_chordal_batch(host, 512)
    assert (orders == o).all() and (wit == w).all()
    # unpadded host rows (row_bytes = ceil(n/8) < device stride)
    g = [gen_chordal_random(100, 4, s) for s in range(5)]
    h2 = np.stack([x._packed for x in g])
    o2 = np.empty((5, 100), dtype=np.int32)
    w2 = np.empty((5, 3), dtype=np.int32)
    assert _native.lib.chordal_is_chordal_batch_host(h2.ctypes.data, 5, 100, 13, o2.ctypes.data, w2.ctypes.data, 2) == 0
    v3, o3, w3 = oracle.is_chordal_batch(h2, 100)
    assert (o2 == o3).all() and (w2 == w3).all()
    # the workspace form (repeated calls): same results, workspace reused
    wsb = int(_native.lib.chordal_batch_host_workspace_bytes(512, 7))
    ws = torch.empty(wsb + 256, dtype=torch.uint8, device="cuda")
    wp = (ws.data_ptr() + 255) & ~255
    for _ in range(2):
        o4 = np.empty((40, 512), dtype=np.int32)
        w4 = np.empty((40, 3), dtype=np.int32)
        assert _native.lib.chordal_is_chordal_batch_host_ws(host.ctypes.data, 40, 512, 64, o4.ctypes.data,
                                                            w4.ctypes.data, 7, wp, wsb) == 0
        assert (o4 == o).all() and (w4 == w).all()
    assert _native.lib.chordal_is_chordal_batch_host_ws(host.ctypes.data, 40, 512, 64, o4.ctypes.data,
                                                        w4.ctypes.data, 7, wp, wsb - 1) == _native.EINVAL
    torch.cuda.synchronize()


def test_host_buffer_entry_point():
    for g in (gen_chordal_random(1000, 8, 0), remove_first_chord(gen_chordal_random(1000, 8, 0))[0],
              gen_dense_random(777, 0.5, 1)):
        n = g.n
        order = np.empty(n, dtype=np.int32)
        wit = np.empty(3, dtype=np.int32)
        chordal = ctypes.c_int32(-1)
        packed = np.ascontiguousarray(g._packed)
        rc = _native.lib.chordal_is_chordal_dense_host(
            packed.ctypes.data, n, packed.shape[1], 0, 0, order.ctypes.data, wit.ctypes.data, ctypes.byref(chordal))
        assert rc == 0
        ok, o, w = oracle.is_chordal(packed, n)
        assert bool(chordal.value) == ok and order.tolist() == o.tolist()
        assert (wit.tolist() if not ok else None) == (None if w is None else list(w))


def test_host_buffer_workspace_entry_point():
    """chordal_is_chordal_dense_host_ws: one workspace reused across graphs of the
    three engine ranges (warp n <= 1024, CTA n <= 32768, CSR beyond)."""
    import torch

    graphs = [gen_chordal_random(1000, 8, 0), remove_first_chord(gen_chordal_random(1000, 8, 0))[0],
              gen_chordal_random(3000, 20, 2), gen_dense_random(2500, 0.4, 3),
              gen_chordal_random(33000, 3, 4, cap=33000)]
    big = max(int(_native.lib.chordal_dense_host_workspace_bytes(g.n, g.m)) for g in graphs)
    ws = torch.empty(big + 256, dtype=torch.uint8, device="cuda")
    wp = (ws.data_ptr() + 255) & ~255
    for g in graphs:
        n = g.n
        order = np.empty(n, dtype=np.int32)
        wit = np.empty(3, dtype=np.int32)
        chordal = ctypes.c_int32(-1)
        packed = np.ascontiguousarray(g._packed)
        rc = _native.lib.chordal_is_chordal_dense_host_ws(packed.ctypes.data, n, packed.shape[1], g.m, 0, 0,
                                                          order.ctypes.data, wit.ctypes.data, ctypes.byref(chordal),
                                                          wp, big)
        assert rc == 0
        ok, o, w = oracle.is_chordal(packed, n)
        assert bool(chordal.value) == ok and order.tolist() == o.tolist(), n
        assert (wit.tolist() if not ok else None) == (None if w is None else list(w)), n


def test_reference_graph_objects_are_accepted():
    """Any object with n and _packed (e.g. a chordalkit.Graph) is a valid input."""

    class Foreign:
        __slots__ = ("n", "_packed", "m")

        def __init__(self, g):
            self.n, self._packed, self.m = g.n, g._packed, g.m

        def has_edge(self, u, v):
            return bool((self._packed[u - 1, (v - 1) >> 3] >> ((v - 1) & 7)) & 1)

    g = remove_first_chord(gen_chordal_random(300, 5, 1))[0]
    f = Foreign(g)
    v = P.is_chordal(f)
    assert not v.chordal and v.witness.verify(f, P.lexbfs_partition(f))
    assert w0(v.witness) == w0(P.is_chordal(g).witness)


def test_edge_cases():
    e0 = P.Graph.from_edge_list(0, [])
    v = P.is_chordal(e0)
    assert v.chordal and list(v.peo) == []
    assert P.is_peo(e0, P.VertexOrdering([])) == (True, None)
    assert list(P.is_chordal(P.Graph.from_edge_list(1, [])).peo) == [1]
    assert list(P.parallel_lexbfs(P.Graph.from_edge_list(2, [(1, 2)]), ASC)) == [1, 2]
    big = P.Graph.from_edge_list(32768, [], cap=32768)
    assert o0(P.lexbfs_partition(big)) == list(range(32768))
    assert o0(P.parallel_lexbfs(big, DESC)) == [0] + list(range(32767, 0, -1))
    star = P.Graph.from_edge_list(32768, [(1, k) for k in range(2, 32769)], cap=32768)
    v = P.is_chordal(star)
    assert v.chordal and o0(v.peo) == list(range(32768))
    # sparse graphs beyond the arrangement kernel's SMEM capacity take the slot engine
    assert o0(P.lexbfs_partition(P.Graph.from_edge_list(32769, [], cap=40000))) == list(range(32769))
    # dense graphs beyond it too (CSR slot engine, early exit once classes are singletons)
    dense = P.Graph._from_packed(32800, gen_dense_random_device(32800, 0.5, 1)[0, :, :4100].cpu().numpy(),)
    ok, order, w = oracle.is_chordal(dense._packed, 32800)
    v = P.is_chordal(dense)
    assert not ok and not v.chordal and w0(v.witness) == list(w)
    assert o0(P.lexbfs_partition(dense)) == order.tolist()
    with pytest.raises(P.GraphTooLarge):
        P.is_chordal_batch([P.Graph.from_edge_list(1025, [])])


# ------------------------------------------------------------------- CSR ----


def _csr_cases():
    from paper_1508_06329_b200.csr import CSRGraph
    from paper_1508_06329_b200.generate import chordal_random_edges

    out = []
    for n, k, seed in ((50, 3, 1), (700, 8, 2), (5000, 8, 3), (20000, 4, 4)):
        u, v = chordal_random_edges(n, k, seed)
        out.append((f"chordal{n}", CSRGraph.from_edges0(n, u, v)))
        g = CSRGraph.from_edges0(n, u, v)
        h, _ = remove_first_chord(P.Graph._from_packed(n, gen_chordal_random(n, k, seed, cap=n)._packed)) \
            if n <= 5000 else (None, None)
        if h is not None:
            out.append((f"chordal{n}-chord", CSRGraph.from_dense(h)))
    for n, p, seed in ((300, 0.02, 5), (3000, 0.002, 6)):
        out.append((f"sparse{n}", CSRGraph.from_dense(gen_dense_random(n, p, seed))))
    return out


@pytest.mark.parametrize("name,g", _csr_cases(), ids=[c[0] for c in _csr_cases()])
def test_csr_against_oracle(name, g):
    n = g.n
    order = oracle.lexbfs_partition_csr(g.indptr, g.indices, n)
    ok, w = oracle.is_peo_csr(g.indptr, g.indices, n, order)
    assert o0(P.lexbfs_partition(g)) == order.tolist()
    v = P.is_chordal(g)
    assert v.chordal == ok and w0(v.witness) == (None if w is None else list(w))
    perm = np.random.default_rng(n).permutation(n)
    ok2, w2 = oracle.is_peo_csr(g.indptr, g.indices, n, perm)
    okg, wg = P.is_peo(g, P.VertexOrdering.from_zero_based(perm))
    assert okg == ok2 and w0(wg) == (None if w2 is None else list(w2))
    if n <= 5000:  # the arbitrated rules against the dense oracle
        from paper_1508_06329_b200.graph import row_width

        rows = np.zeros((n, n), dtype=bool)
        for a in range(n):
            rows[a, g.indices[g.indptr[a]:g.indptr[a + 1]]] = True
        packed = np.packbits(rows, axis=1, bitorder="little")
        for arb, mode, seed in ((DESC, oracle.ARB_DESCENDING, 0), (Arbitration.seeded(3), oracle.ARB_SEEDED, 3)):
            assert o0(P.parallel_lexbfs(g, arb)) == oracle.lexbfs_arbitrated(packed, n, mode, seed).tolist()
        assert packed.shape[1] == row_width(n)


def test_dense_to_csr_roundtrip():
    from paper_1508_06329_b200 import ops
    from paper_1508_06329_b200.csr import CSRGraph

    for g in (gen_chordal_random(3000, 8, 1), gen_dense_random(777, 0.3, 2), P.Graph.from_edge_list(5, [])):
        from paper_1508_06329_b200.device import device_rows

        ip, ix = ops.dense_to_csr(device_rows(g))
        ref = CSRGraph.from_dense(g)
        assert ip.cpu().numpy().tolist() == ref.indptr.tolist()
        assert ix.cpu().numpy().tolist() == ref.indices.tolist()


@pytest.mark.slow
@pytest.mark.skipif("5" not in CONFIGS, reason="configs.json not generated")
def test_config5_csr_million():
    from paper_1508_06329_b200.csr import CSRGraph
    from paper_1508_06329_b200.generate import chordal_random_edges

    from paper_1508_06329_b200.generate import gen_chordal_random_csr_device

    exp = CONFIGS["5"]
    ip, ix = gen_chordal_random_csr_device(exp["n"], exp["k"], exp["seed"])  # drawn on the GPU
    g = CSRGraph(exp["n"], ip.cpu().numpy(), ix.cpu().numpy())
    assert sha(g.indptr) == exp["indptr_sha256"] and sha(g.indices) == exp["indices_sha256"]
    u = np.repeat(np.arange(g.n), np.diff(g.indptr))
    v = g.indices.astype(np.int64)
    keep0 = u < v
    u, v = u[keep0], v[keep0]
    vd = P.is_chordal(g)
    assert vd.chordal and sha(vd.peo.order0.astype(np.int32)) == exp["order_sha256"]
    a, b = exp["nonchordal"]["removed_edge0"]
    keep = ~(((u == a) & (v == b)) | ((u == b) & (v == a)))
    h = CSRGraph.from_edges0(exp["n"], u[keep], v[keep])
    vn = P.is_chordal(h)
    assert not vn.chordal and w0(vn.witness) == exp["nonchordal"]["witness"]
    assert sha(P.lexbfs_partition(h).order0.astype(np.int32)) == exp["nonchordal"]["order_sha256"]


def test_device_csr_generator_matches_host():
    from paper_1508_06329_b200.csr import CSRGraph
    from paper_1508_06329_b200.generate import chordal_random_edges, gen_chordal_random_csr_device

    for n, k, seed in ((2000, 8, 3), (500, 30, 1), (64, 0, 2), (1, 0, 0)):
        ip, ix = gen_chordal_random_csr_device(n, k, seed)
        u, v = chordal_random_edges(n, k, seed)
        ref = CSRGraph.from_edges0(n, u, v)
        assert ip.cpu().numpy().tolist() == ref.indptr.tolist()
        assert ix.cpu().numpy().tolist() == ref.indices.tolist()


# ------------------------------------------------- seeded linked variants ----


def test_seeded_linked_goldens():
    """lexbfs_partition / lexbfs_labels with seeded(s), method="linked" (and
    "auto" below 1024 vertices): the reference's frozen orders, and is_chordal
    with method="reference" (tests/golden/seeded_linked.npz)."""
    z = load_npz("seeded_linked.npz")
    for i in range(len(z["n"])):
        n, s = int(z["n"][i]), int(z["seed"][i])
        g = G(z["packed"][i, :n, : (n + 7) // 8], n)
        assert o0(P.lexbfs_partition(g, P.seeded(s), method="linked")) == z["part"][i, :n].tolist(), i
        assert o0(P.lexbfs_labels(g, P.seeded(s), method="linked")) == z["labels"][i, :n].tolist(), i
        if n < 1024:
            assert o0(P.lexbfs_partition(g, P.seeded(s))) == z["part"][i, :n].tolist(), i
        v = P.is_chordal(g, "partition", P.seeded(s), method="reference")
        assert bool(v.chordal) == bool(z["chordal"][i]), i
        assert (w0(v.witness) or [-1, -1, -1]) == z["witness"][i].tolist(), i


def test_seeded_linked_against_oracle_larger():
    from paper_1508_06329_b200.csr import CSRGraph

    cases = [gen_chordal_random(3000, 12, 5), gen_dense_random(2500, 0.01, 6), gen_dense_random(1200, 0.6, 7),
             gen_chordal_random(40000, 6, 8, cap=40000)]
    for k, g in enumerate(cases):
        for s in (0, 77 + k, -3):
            for variant, fn in (("partition", P.lexbfs_partition), ("labels", P.lexbfs_labels)):
                want = oracle.lexbfs_linked_seeded(g._packed, g.n, s, variant).tolist()
                assert o0(fn(g, P.seeded(s), method="linked")) == want, (k, s, variant)
    # CSR input (the N > 32768 global-memory slot engine)
    from paper_1508_06329_b200.generate import chordal_random_edges

    g = cases[-1]
    u, v = chordal_random_edges(40000, 6, 8)
    c = CSRGraph.from_edges0(g.n, u, v)
    want = oracle.lexbfs_linked_seeded(g._packed, g.n, 9, "labels").tolist()
    assert o0(P.lexbfs_labels(c, P.seeded(9), method="linked")) == want


# ------------------------------------------------ MCS and BFS orderings ----


def test_mcs_bfs_goldens():
    """mcs_order / bfs_order (search.py:79-145): the reference's frozen orders,
    LOWEST_INDEX and seeded, plus its named cases (test_search.py:53-66)."""
    z = load_npz("seeded_linked.npz")
    for i in range(len(z["n"])):
        n, s = int(z["n"][i]), int(z["seed"][i])
        g = G(z["packed"][i, :n, : (n + 7) // 8], n)
        if z["mcs"][i, 0] >= 0 or n == 0:
            assert o0(P.mcs_order(g)) == z["mcs"][i, :n].tolist(), i
            assert o0(P.mcs_order(g, P.seeded(s))) == z["mcs_seeded"][i, :n].tolist(), i
        assert o0(P.bfs_order(g)) == z["bfs"][i, :n].tolist(), i
        assert o0(P.bfs_order(g, P.seeded(s))) == z["bfs_seeded"][i, :n].tolist(), i
    c4 = P.Graph.from_edge_list(4, [(1, 2), (2, 3), (3, 4), (4, 1)])
    assert list(P.bfs_order(c4)) == [1, 2, 4, 3] and list(P.mcs_order(c4)) == [1, 2, 3, 4]
    assert list(P.bfs_order(P.Graph.from_edge_list(4, [(1, 2), (3, 4)]))) == [1, 2, 3, 4]
    star = P.Graph.from_edge_list(5, [(1, k) for k in range(2, 6)])
    assert list(P.mcs_order(star)) == [1, 2, 3, 4, 5]


def test_mcs_bfs_against_oracle_larger():
    """Larger graphs vs the oracle; MCS + is_peo decides chordality (Tarjan-Yannakakis,
    the reference's test_peo.py:127-129)."""
    from paper_1508_06329_b200.csr import CSRGraph
    from paper_1508_06329_b200.generate import chordal_random_edges

    for k, g in enumerate([gen_chordal_random(3000, 10, 11), gen_dense_random(2000, 0.3, 12),
                           gen_dense_random(5000, 0.002, 13)]):
        for s in (None, 5 + k):
            tb = P.LOWEST_INDEX if s is None else P.seeded(s)
            assert o0(P.mcs_order(g, tb)) == oracle.other_order(g._packed, g.n, "mcs", s).tolist(), (k, s)
            assert o0(P.bfs_order(g, tb)) == oracle.other_order(g._packed, g.n, "bfs", s).tolist(), (k, s)
        ok, _ = P.is_peo(g, P.mcs_order(g))
        assert ok == P.is_chordal(g).chordal
    u, v = chordal_random_edges(200000, 6, 3)
    c = CSRGraph.from_edges0(200000, u, v)
    got = P.bfs_order(c).order0
    assert sorted(got.tolist()) == list(range(200000)) and got[0] == 0


def test_csr_peo_heavy_rows():
    """Rows longer than the heavy threshold (4096) are checked by the whole grid:
    a hub with 9000 neighbours on a chordless 4-cycle, LexBFS order and random
    orders (parents searched), against the oracle's list PEO test."""
    from paper_1508_06329_b200.csr import CSRGraph

    rng = np.random.default_rng(11)
    n = 12000
    us, vs = [0, 1, 2, 3], [1, 2, 3, 0]                    # C4: 0-1-2-3-0, no 0-2, no 1-3
    hub = [w for w in range(4, 9004)]
    us += [0] * len(hub)
    vs += hub
    a = rng.integers(4, n, 20000)
    b = rng.integers(4, n, 20000)
    keep = a != b
    us += a[keep].tolist()
    vs += b[keep].tolist()
    g = CSRGraph.from_edges0(n, np.array(us), np.array(vs))
    ip, ix = g.indptr, g.indices
    v = P.is_chordal(g)
    order = oracle.lexbfs_partition_csr(ip, ix, n)
    ok, w = oracle.is_peo_csr(ip, ix, n, order)
    assert v.chordal == ok and o0(P.lexbfs_partition(g)) == order.tolist()
    assert (w0(v.witness) or [-1, -1, -1]) == (list(w) if w is not None else [-1, -1, -1])
    for s in range(3):
        perm = rng.permutation(n).astype(np.int32)
        ok2, w2 = oracle.is_peo_csr(ip, ix, n, perm)
        okg, wg = P.is_peo(g, P.VertexOrdering.from_zero_based(perm))
        assert okg == ok2 and (w0(wg) or [-1, -1, -1]) == (list(w2) if w2 is not None else [-1, -1, -1]), s
    # chordal with a heavy hub: star + random tree edges between leaves' private vertices
    us2 = [0] * 8000 + list(range(8001, 11000))
    vs2 = list(range(1, 8001)) + [int(x) for x in rng.integers(1, 8001, 2999)]
    g2 = CSRGraph.from_edges0(11000, np.array(us2), np.array(vs2))
    order2 = oracle.lexbfs_partition_csr(g2.indptr, g2.indices, 11000)
    ok3, _ = oracle.is_peo_csr(g2.indptr, g2.indices, 11000, order2)
    assert P.is_chordal(g2).chordal == ok3


def test_new_orderings_edge_cases():
    """n = 0 / 1 / edgeless / complete for MCS, BFS and the seeded linked variants."""
    from paper_1508_06329_b200.csr import CSRGraph

    for n in (0, 1, 2, 7):
        e = P.Graph.from_edge_list(n, [])
        k = P.Graph.from_edge_list(n, [(a, b) for a in range(1, n + 1) for b in range(a + 1, n + 1)])
        for g in (e, k):
            want = list(range(1, n + 1))
            assert list(P.mcs_order(g)) == want and list(P.bfs_order(g)) == want
            assert list(P.lexbfs_partition(g, P.seeded(3), method="linked")) == \
                [x + 1 for x in oracle.lexbfs_linked_seeded(g._packed, n, 3, "partition").tolist()]
            assert list(P.lexbfs_labels(g, P.seeded(3), method="linked")) == \
                [x + 1 for x in oracle.lexbfs_linked_seeded(g._packed, n, 3, "labels").tolist()]
            assert list(P.mcs_order(g, P.seeded(5))) == [x + 1 for x in oracle.other_order(g._packed, n, "mcs", 5)]
            assert list(P.bfs_order(g, P.seeded(5))) == [x + 1 for x in oracle.other_order(g._packed, n, "bfs", 5)]
    c = CSRGraph.from_edges0(3, np.array([0]), np.array([2]))
    assert list(P.bfs_order(c)) == [1, 3, 2]


@pytest.mark.gpu
@pytest.mark.parametrize("n", [8000, 40000])
def test_csr_global_engine_tie_rules_and_components(n):
    """The global-memory slot engine (CSR, n > 32768) with its <= 32-neighbour fast
    step: LOWEST_INDEX against the oracle's PartitionList, and the descending rule
    through the relabelling v -> n - v (v >= 1) that turns it into LOWEST_INDEX
    (the initial class [1, n, n-1, ..., 2] of parallel/lexbfs.py:173 becomes
    ascending); graphs with many components exercise the new-component steps."""
    from paper_1508_06329_b200.csr import CSRGraph
    from paper_1508_06329_b200.generate import chordal_random_edges

    # n = 8000: the all-in-shared-memory slot kernel (u16 slots, compaction runs:
    # its slot array holds fewer than n + m slots); n = 40000: the global-memory one
    rng = np.random.default_rng(1508)
    cases = []
    u, v = chordal_random_edges(n, 6, 11)
    cases.append(("chordal", u, v))
    a = rng.integers(0, n, 3 * n // 4)
    b = rng.integers(0, n, 3 * n // 4)
    keep = a != b
    cases.append(("forest-ish", a[keep], b[keep]))
    hub = np.zeros(5000, dtype=np.int64) + 7  # one vertex with > 32 neighbours among small ones
    cases.append(("hub", np.concatenate([a[keep], hub]), np.concatenate([b[keep], rng.integers(0, n, 5000)])))
    relabel = np.concatenate([[0], n - np.arange(1, n)])  # f(0) = 0, f(v) = n - v
    for name, uu, vv in cases:
        lo, hi = np.minimum(uu, vv), np.maximum(uu, vv)
        pairs = np.unique(np.stack([lo, hi], 1)[lo != hi], axis=0)
        g = CSRGraph.from_edges0(n, pairs[:, 0], pairs[:, 1])
        want = oracle.lexbfs_partition_csr(g.indptr, g.indices, n)
        assert o0(P.lexbfs_partition(g)) == want.tolist(), name
        ok, w = oracle.is_peo_csr(g.indptr, g.indices, n, want)
        verdict = P.is_chordal(g)
        assert verdict.chordal == ok and w0(verdict.witness) == (None if w is None else list(w)), name
        gr = CSRGraph.from_edges0(n, relabel[pairs[:, 0]], relabel[pairs[:, 1]])
        want_desc = relabel[oracle.lexbfs_partition_csr(gr.indptr, gr.indices, n)]  # f is an involution
        assert o0(P.parallel_lexbfs(g, DESC)) == want_desc.tolist(), name
        if n <= 16384:  # seeded arbitration against the dense oracle
            packed = np.zeros((n, (n + 7) // 8), dtype=np.uint8)
            for x, y in ((pairs[:, 0], pairs[:, 1]), (pairs[:, 1], pairs[:, 0])):
                np.bitwise_or.at(packed, (x, y >> 3), (1 << (y & 7)).astype(np.uint8))
            want_arb = oracle.lexbfs_arbitrated(packed, n, oracle.ARB_SEEDED, 3).tolist()
            assert o0(P.parallel_lexbfs(g, Arbitration.seeded(3))) == want_arb, name
