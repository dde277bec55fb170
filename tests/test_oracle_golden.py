"""Pin the CPU oracle (oracle/chordal_oracle.c) to the reference's own outputs.

Every fixture under tests/golden/ was produced by running the reference
package (tests/golden/make_golden.py); the oracle must reproduce each one
exactly before it is trusted as the checker of the CUDA path.
"""

import hashlib

import numpy as np
import pytest

import oracle
from conftest import exhaustive_graph_packed, load_json, load_npz, named_packed


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


NAMED = load_json("named.json")


@pytest.mark.parametrize("rec", NAMED["graphs"], ids=[r["name"] for r in NAMED["graphs"]])
def test_oracle_named(rec):
    n = rec["n"]
    packed = named_packed(rec)
    assert oracle.lexbfs_partition(packed, n).tolist() == rec["lexbfs_partition"]
    assert oracle.lexbfs_array(packed, n).tolist() == rec["lexbfs_labels"]
    assert oracle.lexbfs_arbitrated(packed, n, oracle.ARB_ASCENDING).tolist() == rec["par_asc"]
    assert oracle.lexbfs_arbitrated(packed, n, oracle.ARB_DESCENDING).tolist() == rec["par_desc"]
    for s, o in rec["par_seeded"].items():
        assert oracle.lexbfs_arbitrated(packed, n, oracle.ARB_SEEDED, int(s)).tolist() == o
    ok, order, w = oracle.is_chordal(packed, n)
    assert ok == rec["chordal"]
    assert (None if w is None else list(w)) == rec["witness"]
    o6 = oracle.lexbfs_arbitrated(packed, n, oracle.ARB_SEEDED, 6)
    ok6, w6 = oracle.is_peo(packed, n, o6)
    assert ok6 == rec["par_seeded6_chordal"]
    assert (None if w6 is None else list(w6)) == rec["par_seeded6_witness"]


def test_oracle_frozen_peo_cases():
    graphs = {r["name"]: r for r in NAMED["graphs"]}
    for case in NAMED["peo_cases"]:
        rec = graphs[case["graph"]]
        ok, w = oracle.is_peo(named_packed(rec), rec["n"], np.array(case["order"]))
        assert ok == case["ok"]
        assert (None if w is None else list(w)) == case["witness"]


def test_oracle_frozen_reference_values():
    """The literal goldens of the reference suite."""
    graphs = {r["name"]: r for r in NAMED["graphs"]}
    c4 = graphs["c4"]
    assert [v + 1 for v in oracle.lexbfs_partition(named_packed(c4), 4)] == [1, 2, 4, 3]
    assert [v + 1 for v in oracle.lexbfs_arbitrated(named_packed(c4), 4, oracle.ARB_DESCENDING)] == [1, 4, 2, 3]
    ok, w = oracle.is_peo(named_packed(c4), 4, np.array([0, 1, 3, 2]))
    assert not ok and tuple(x + 1 for x in w) == (3, 4, 2)
    p3r = graphs["p3_relabeled"]
    assert [v + 1 for v in oracle.lexbfs_partition(named_packed(p3r), 3)] == [1, 3, 2]
    d6 = graphs["disconnected6"]
    assert [v + 1 for v in oracle.lexbfs_partition(named_packed(d6), 6)] == [1, 3, 2, 5, 6, 4]


def test_oracle_random_small(small_corpus):
    c = small_corpus
    for i in range(len(c)):
        n = int(c.ns[i])
        P = c.packed(i)
        assert oracle.lexbfs_partition(P, n).tolist() == c.vec("lex", i).tolist(), i
        assert oracle.lexbfs_array(P, n).tolist() == c.vec("lex", i).tolist(), i
        assert oracle.lexbfs_arbitrated(P, n, oracle.ARB_DESCENDING).tolist() == c.vec("par_desc", i).tolist()
        assert oracle.lexbfs_arbitrated(P, n, oracle.ARB_SEEDED, i).tolist() == c.vec("par_seeded", i).tolist()
        from paper_1508_06329_b200.generate import stream

        init = stream(i, "lexbfs-partition").permutation(n)
        assert oracle.lexbfs_array(P, n, init).tolist() == c.vec("seeded_array", i).tolist()
        ok, w = oracle.is_peo(P, n, c.vec("perm", i))
        assert ok == bool(c.z["perm_ok"][i])
        assert (list(w) if w else [-1, -1, -1]) == c.z["perm_witness"][i].tolist()
        ok2, _, w2 = oracle.is_chordal(P, n)
        assert (list(w2) if w2 else [-1, -1, -1]) == c.z["chordal_witness"][i].tolist()


def test_oracle_exhaustive5():
    z = load_npz("exhaustive5.npz")
    for k in range(len(z["n"])):
        n, mask = int(z["n"][k]), int(z["mask"][k])
        P = exhaustive_graph_packed(n, mask)
        ok, order, w = oracle.is_chordal(P, n)
        assert order.tolist() == z["order"][k][:n].tolist()
        assert ok == bool(z["chordal"][k])
        assert (list(w) if w else [-1, -1, -1]) == z["witness"][k].tolist()


def test_oracle_csr_matches_dense(small_corpus):
    c = small_corpus
    for i in range(0, len(c), 3):
        n = int(c.ns[i])
        rows = np.unpackbits(c.packed(i), axis=1, bitorder="little", count=n).astype(bool)
        indptr = np.concatenate([[0], np.cumsum(rows.sum(axis=1))]).astype(np.int64)
        indices = np.flatnonzero(rows.reshape(-1)) % max(n, 1)
        assert oracle.lexbfs_partition_csr(indptr, indices, n).tolist() == c.vec("lex", i).tolist()
        ok, w = oracle.is_peo_csr(indptr, indices, n, c.vec("perm", i))
        assert ok == bool(c.z["perm_ok"][i])
        assert (list(w) if w else [-1, -1, -1]) == c.z["perm_witness"][i].tolist()


CONFIGS = load_json("configs.json") if __import__("os").path.exists(
    __import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "configs.json")) else {}


@pytest.mark.skipif("1" not in CONFIGS, reason="configs.json not generated")
def test_oracle_config1():
    from paper_1508_06329_b200.generate import gen_chordal_random, packed_sha256, remove_first_chord

    orders = load_npz("configs_orders.npz")
    g = gen_chordal_random(1000, 8, 0)
    h, e = remove_first_chord(g)
    for graph, key, ok_key in ((g, "chordal", "c1_chordal"), (h, "nonchordal", "c1_nonchordal")):
        exp = CONFIGS["1"][key]
        assert packed_sha256(graph._packed) == exp["packed_sha256"]
        ok, order, w = oracle.is_chordal(graph._packed, 1000)
        assert order.tolist() == orders[ok_key].astype(int).tolist()
        assert ok == exp["chordal"]
        assert (None if w is None else list(w)) == exp["witness"]
    assert list(e) == CONFIGS["1"]["nonchordal"]["removed_edge"]


@pytest.mark.skipif("4" not in CONFIGS, reason="configs.json not generated")
def test_oracle_config4_sample():
    from paper_1508_06329_b200.generate import gen_chordal_random, gen_dense_random, packed_sha256

    for rec in CONFIGS["4"]["sample"][:24]:
        s = rec["seed"]
        g = gen_dense_random(512, 0.5, s) if s % 2 == 0 else gen_chordal_random(512, 8, s)
        assert packed_sha256(g._packed) == rec["packed_sha256"]
        ok, order, w = oracle.is_chordal(g._packed, 512)
        assert _sha(order.astype(np.int32)) == rec["order_sha256"]
        assert ok == rec["chordal"]
        assert (None if w is None else list(w)) == rec["witness"]


def test_oracle_batch_matches_single(small_corpus):
    from paper_1508_06329_b200.generate import gen_chordal_random, gen_dense_random

    gs = [gen_dense_random(96, 0.4, s) if s % 2 == 0 else gen_chordal_random(96, 4, s) for s in range(12)]
    adj = np.stack([g._packed for g in gs])
    verdict, orders, wit = oracle.is_chordal_batch(adj, 96, nthreads=3)
    for b, g in enumerate(gs):
        ok, order, w = oracle.is_chordal(g._packed, 96)
        assert verdict[b] == ok and orders[b].tolist() == order.tolist()
        assert (list(w) if w else [-1, -1, -1]) == wit[b].tolist()


def test_oracle_seeded_linked_goldens():
    """Seeded linked LexBFS (search.py:283-310, 515-532) with the C Philox port:
    the orders the reference produced (tests/golden/seeded_linked.npz)."""
    z = load_npz("seeded_linked.npz")
    for i in range(len(z["n"])):
        n, s = int(z["n"][i]), int(z["seed"][i])
        rows = z["packed"][i, :n, : (n + 7) // 8]
        assert oracle.lexbfs_linked_seeded(rows, n, s, "partition").tolist() == z["part"][i, :n].tolist(), i
        assert oracle.lexbfs_linked_seeded(rows, n, s, "labels").tolist() == z["labels"][i, :n].tolist(), i


def test_oracle_mcs_bfs_goldens():
    """mcs_order / bfs_order (search.py:79-145), LOWEST_INDEX and seeded: the
    reference's frozen orders (tests/golden/seeded_linked.npz; MCS for n <= 400)."""
    z = load_npz("seeded_linked.npz")
    for i in range(len(z["n"])):
        n, s = int(z["n"][i]), int(z["seed"][i])
        rows = z["packed"][i, :n, : (n + 7) // 8]
        if z["mcs"][i, 0] >= 0 or n == 0:
            assert oracle.other_order(rows, n, "mcs").tolist() == z["mcs"][i, :n].tolist(), i
            assert oracle.other_order(rows, n, "mcs", s).tolist() == z["mcs_seeded"][i, :n].tolist(), i
        assert oracle.other_order(rows, n, "bfs").tolist() == z["bfs"][i, :n].tolist(), i
        assert oracle.other_order(rows, n, "bfs", s).tolist() == z["bfs_seeded"][i, :n].tolist(), i


def test_oracle_lexbfs_certificate_on_reference_orders(small_corpus):
    """The certificate (oracle.lexbfs_certify) accepts every LexBFS order the
    reference produced -- LOWEST_INDEX exactly, the descending / seeded
    arbitration and seeded-array orders as LexBFS orders that leave the
    LOWEST_INDEX choice at their first difference from it -- and rejects
    non-LexBFS orders (the random permutations) at a step where a smaller label
    was taken."""
    c = small_corpus
    rejected = 0
    for i in range(0, len(c), 3):
        n = int(c.ns[i])
        P = c.packed(i)
        lex = c.vec("lex", i).tolist()
        assert oracle.lexbfs_certify(P, n, lex) == (-1, -1), i
        for key in ("par_desc", "par_seeded", "seeded_array"):
            o = c.vec(key, i).tolist()
            first = next((k for k in range(n) if o[k] != lex[k]), -1)
            assert oracle.lexbfs_certify(P, n, o) == (-1, first), (i, key)
        bad, off = oracle.lexbfs_certify(P, n, c.vec("perm", i).tolist())
        if bad >= 0:
            rejected += 1
            assert 0 < bad and off <= bad
    assert rejected > 0
