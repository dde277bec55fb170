"""Fixtures frozen from the reference for left neighbourhoods, ScanStats and the
large seeded tie rules.

Run in the development container (the reference is importable only here):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_left_golden.py [left|seeded|all]

Outputs (committed):
  left_scan.npz   600 (graph, ordering) cases: the reference's
                  left_neighborhoods(g, o) parents and |LN(v)| (graph.py:284-302),
                  is_peo(g, o, stats=ScanStats()) verdict, witness and the
                  list scan's reads / budget (peo.py:100-149).  Orderings
                  alternate between the LexBFS order and a random permutation
                  (so both PEO and non-PEO scans are pinned).
  seeded_large.npz  lexbfs_partition(g, seeded(s), method="array") orders at
                  n = 2048 and n = 8192 (search.py:535-541, the seeded path the
                  reference takes for n >= 1024), and
                  parallel_lexbfs(g, Arbitration.seeded(s)) at n = 40000 (the
                  dense-stored graph that runs on the global slot engine), with
                  the reference's wall times.
"""

from __future__ import annotations

import os
import random
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import chordalkit as C  # noqa: E402
from chordalkit.graph import left_neighborhoods  # noqa: E402
from chordalkit.parallel import Arbitration, parallel_lexbfs  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(OUT))
sys.path.insert(0, ROOT)


def wit0(w):
    return [-1, -1, -1] if w is None else [w.v - 1, w.p - 1, w.z - 1]


def _graph(rng: random.Random, s: int):
    n = rng.choice([1, 2, 3, 4, 6, 9, 16, 31, 32, 33, 48, 64, 65, 100, 128, 150, 200, 257])
    kind = s % 4
    if n < 3 or kind == 0:
        p = (0.1, 0.25, 0.5, 0.75, 0.9)[s % 5]
        return C.gen_dense_random(n, p, s) if n > 1 else C.Graph.from_edge_list(1, [])
    g = C.gen_chordal_random(n, min(n - 1, 1 + s % 7), s)
    if kind == 3 and n > 4:
        from paper_1508_06329_b200.generate import remove_first_chord  # noqa: E402

        h, _ = remove_first_chord(C.Graph(g.n, g._packed.copy(), g.m))
        g = C.Graph(h.n, np.array(h._packed), h.m)
    if kind == 2 and n >= 41:  # sparse random (not chordal in general)
        g = C.gen_sparse_random(n, s)
    return g


def make_left(count: int = 600):
    rng = random.Random(1508_0629)
    ns, packed, offs, orders, parents, lnsz = [], [], [0], [], [], []
    ok, wit, reads, budget = [], [], [], []
    for s in range(count):
        g = _graph(rng, s)
        n = g.n
        if s % 2 == 0:
            o = C.lexbfs_partition(g)
        else:
            perm = list(range(1, n + 1))
            rng.shuffle(perm)
            o = C.VertexOrdering(perm)
        ln = left_neighborhoods(g, o)
        st = C.ScanStats()
        k, w = C.is_peo(g, o, stats=st)
        ns.append(n)
        packed.append(np.asarray(g._packed).reshape(-1))
        offs.append(offs[-1] + g._packed.size)
        orders.append([v - 1 for v in o])
        parents.append([(ln.parent(v) or 0) - 1 for v in range(1, n + 1)])
        lnsz.append([len(ln.ln(v)) for v in range(1, n + 1)])
        ok.append(k)
        wit.append(wit0(w))
        reads.append(st.reads)
        budget.append(st.budget)
    flat = lambda xs: np.array([x for row in xs for x in row], dtype=np.int32)  # noqa: E731
    np.savez_compressed(
        os.path.join(OUT, "left_scan.npz"),
        n=np.array(ns, dtype=np.int32),
        packed=np.concatenate(packed).astype(np.uint8),
        packed_off=np.array(offs, dtype=np.int64),
        order=flat(orders),
        parent=flat(parents),
        ln_size=flat(lnsz),
        ok=np.array(ok, dtype=bool),
        witness=np.array(wit, dtype=np.int32),
        reads=np.array(reads, dtype=np.int64),
        budget=np.array(budget, dtype=np.int64),
    )
    print(f"left_scan.npz: {count} cases, {sum(ok)} PEOs", flush=True)


def make_seeded():
    out = {}
    cases = [
        ("array_chordal2048_s7", lambda: C.gen_chordal_random(2048, 8, 3), 7),
        ("array_dense2048_s5", lambda: C.gen_dense_random(2048, 0.3, 4), 5),
        ("array_chordal8192_s11", lambda: C.gen_chordal_random(8192, 8, 0), 11),
    ]
    for name, mk, seed in cases:
        g = mk()
        t0 = time.perf_counter()
        o = C.lexbfs_partition(g, C.seeded(seed), method="array")
        dt = time.perf_counter() - t0
        out[name] = np.asarray(o.order0, dtype=np.int16)
        out[name + "_seconds"] = np.array(dt)
        print(f"{name}: {dt:.2f}s", flush=True)
    g = C.gen_chordal_random(40000, 4, 2, cap=40000)
    for seed in (3,):
        t0 = time.perf_counter()
        o = parallel_lexbfs(g, Arbitration.seeded(seed))
        dt = time.perf_counter() - t0
        out[f"parseeded_chordal40000_k4_s{seed}"] = np.asarray(o.order0, dtype=np.int32)
        out[f"parseeded_chordal40000_k4_s{seed}_seconds"] = np.array(dt)
        print(f"parallel seeded 40000: {dt:.1f}s", flush=True)
    np.savez_compressed(os.path.join(OUT, "seeded_large.npz"), **out)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("left", "all"):
        make_left()
    if what in ("seeded", "all"):
        make_seeded()
