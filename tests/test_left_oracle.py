"""The oracle's literal list scan (oracle_peo_lists_stats) against the
reference's left_neighborhoods / is_peo(stats=...) outputs frozen in
tests/golden/left_scan.npz (600 cases).  CPU only."""

import numpy as np

import oracle


def test_oracle_list_scan_matches_reference_left_and_stats(left_corpus):
    c = left_corpus
    z = c.z
    for i in range(len(c)):
        n = int(c.ns[i])
        ip, ix = oracle.csr_from_packed(c.packed(i), n)
        ok, w, parent, lnsz, reads = oracle.peo_lists_stats(ip, ix, n, c.vec("order", i))
        assert ok == bool(z["ok"][i]), i
        assert (w or (-1, -1, -1)) == tuple(z["witness"][i].tolist()), i
        assert np.array_equal(parent, c.vec("parent", i)), i
        assert np.array_equal(lnsz, c.vec("ln_size", i)), i
        assert reads == int(z["reads"][i]), (i, reads, int(z["reads"][i]))
        assert int(z["budget"][i]) == 8 * (int(ip[-1]) // 2)
        # and the dense list test agrees on verdict and witness
        okd, wd = oracle.is_peo(c.packed(i), n, c.vec("order", i))
        assert okd == ok and wd == w, i


def test_left_corpus_covers_both_outcomes(left_corpus):
    z = left_corpus.z
    assert len(left_corpus) == 600
    assert 100 < int(z["ok"].sum()) < 500
    assert int(left_corpus.ns.max()) >= 200


def test_oracle_seeded_paths_match_reference_large():
    """The oracle's lexbfs_array / arbitrated LexBFS against the reference's frozen
    seeded orders at n = 2048, 8192 and 40000 (seeded_large.npz)."""
    import paper_1508_06329_b200 as P
    from conftest import load_npz
    from paper_1508_06329_b200.generate import gen_chordal_random, gen_dense_random

    z = load_npz("seeded_large.npz")
    for name, g, seed in (("array_chordal2048_s7", gen_chordal_random(2048, 8, 3), 7),
                          ("array_dense2048_s5", gen_dense_random(2048, 0.3, 4), 5),
                          ("array_chordal8192_s11", gen_chordal_random(8192, 8, 0), 11)):
        initial = P.seeded(seed).generator("lexbfs-partition").permutation(g.n)
        assert np.array_equal(oracle.lexbfs_array(g._packed, g.n, initial), z[name].astype(np.int64)), name
    g = gen_chordal_random(40000, 4, 2, cap=40000)
    assert np.array_equal(oracle.lexbfs_arbitrated(g._packed, g.n, oracle.ARB_SEEDED, 3),
                          z["parseeded_chordal40000_k4_s3"])
