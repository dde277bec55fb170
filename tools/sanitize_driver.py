"""Small inputs through every kernel family, for compute-sanitizer runs.

    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python tools/sanitize_driver.py [part]

Parts: warp (one-warp engine, single graph + batch), cta (single-CTA engine,
sparse + dense + seeded arbitration), slot (CSR slot engine, shared-memory and
global-state forms), peo (dense + CSR PEO kernels, heavy rows), other (MCS,
BFS, generators, left neighbourhoods).  Each result is checked against the
oracle (test infrastructure) so a run that passes the sanitizer also passed
parity on the same launch.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1508_06329_b200 as P  # noqa: E402
from paper_1508_06329_b200.csr import CSRGraph  # noqa: E402
from paper_1508_06329_b200.generate import gen_chordal_random, gen_dense_random, remove_first_chord  # noqa: E402


def check_chordal(g):
    v = P.is_chordal(g)
    packed = g._packed if hasattr(g, "_packed") else None
    if packed is not None:
        ok, order, w = oracle.is_chordal(packed, g.n)
    else:
        order = oracle.lexbfs_partition_csr(g.indptr, g.indices, g.n)
        ok, w = oracle.is_peo_csr(g.indptr, g.indices, g.n, order)
    assert v.chordal == ok, "verdict"
    if ok:
        assert v.peo.order0.tolist() == list(order), "order"
    else:
        assert (v.witness.v - 1, v.witness.p - 1, v.witness.z - 1) == tuple(w), "witness"


def part_warp():
    for g in (gen_chordal_random(300, 6, 1), gen_dense_random(200, 0.3, 2)):
        check_chordal(g)
        check_chordal(remove_first_chord(g)[0])
    gs = [gen_dense_random(512, 0.5, s) if s % 2 == 0 else gen_chordal_random(512, 8, s) for s in range(8)]
    bv = P.is_chordal_batch(gs)
    verdict, orders, wit = oracle.is_chordal_batch(np.stack([x._packed for x in gs]), 512)
    assert (bv.chordal == verdict).all() and (bv.orders0 == orders).all() and (bv.witness0 == wit).all()


def part_cta():
    for g in (gen_chordal_random(2500, 16, 3), gen_dense_random(2048, 0.5, 4)):
        check_chordal(g)
        check_chordal(remove_first_chord(g)[0])
    g = gen_chordal_random(1500, 8, 5)
    for arb, mode in ((P.Arbitration.fixed_priority("descending"), 1), (P.Arbitration.seeded(6), 2)):
        o = P.parallel_lexbfs(g, arb)
        ref = oracle.lexbfs_arbitrated(g._packed, g.n, mode, arb.seed or 0)
        assert o.order0.tolist() == ref.tolist(), "arbitrated order"


def part_slot():
    # 3000 / 8000: all state in shared memory (8000: the slot array compacts);
    # 20000: shared-memory class ids, global bookkeeping; 40000: global state
    for n in (8000, 20000):
        from paper_1508_06329_b200.generate import chordal_random_edges

        u, v = chordal_random_edges(n, 6, 7)
        g = CSRGraph.from_edges0(n, u, v)
        check_chordal(g)
        for arb in (P.Arbitration.fixed_priority("descending"), P.Arbitration.seeded(3)):
            assert sorted(P.parallel_lexbfs(g, arb).order0.tolist()) == list(range(n))
    for n in (3000, 40000):
        g = CSRGraph.from_dense(gen_chordal_random(n, 6, 7)) if n <= 3000 else None
        if g is None:
            from paper_1508_06329_b200.generate import chordal_random_edges

            u, v = chordal_random_edges(n, 6, 7)
            g = CSRGraph.from_edges0(n, u, v)
        check_chordal(g)


def part_peo():
    g = gen_chordal_random(3000, 32, 8)
    h, _ = remove_first_chord(g)
    for x in (g, h):
        rng = np.random.default_rng(0)
        perm = rng.permutation(x.n)
        o = P.VertexOrdering.from_zero_based(perm.tolist())
        ok, w = oracle.is_peo(x._packed, x.n, perm)
        want = (ok, None if w is None else tuple(int(t) + 1 for t in w))
        for gg in (x, CSRGraph.from_dense(x)):
            holds, wt = P.is_peo(gg, o)
            assert (holds, None if wt is None else (wt.v, wt.p, wt.z)) == want, "is_peo"
    # a heavy row: a star plus a chordal body
    n = 20000
    from paper_1508_06329_b200.generate import chordal_random_edges

    u, v = chordal_random_edges(n, 4, 9)
    star = np.arange(1, n, dtype=np.int64)
    c = CSRGraph.from_edges0(n, np.concatenate([u, np.zeros(n - 1, np.int64)]), np.concatenate([v, star]))
    check_chordal(c)


def part_other():
    g = gen_chordal_random(700, 8, 10)
    o = P.mcs_order(g)
    assert o.order0.tolist() == oracle.other_order(g._packed, g.n, "mcs").tolist()
    o = P.bfs_order(g)
    assert o.order0.tolist() == oracle.other_order(g._packed, g.n, "bfs").tolist()
    lo = P.lexbfs_partition(g)
    ln = P.left_neighborhoods(g, lo)
    assert len(ln._parent0) == g.n


PARTS = {"warp": part_warp, "cta": part_cta, "slot": part_slot, "peo": part_peo, "other": part_other}

if __name__ == "__main__":
    torch.cuda.set_device(0)
    names = sys.argv[1:] or list(PARTS)
    for name in names:
        PARTS[name]()
        torch.cuda.synchronize()
        print(f"sanitize_driver {name}: ok", flush=True)
