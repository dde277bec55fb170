"""Generate golden fixtures by running the reference package itself.

Run in the development container (the reference is importable only here):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [small|configs|all]

Outputs (committed, small):
  named.json          named graphs of the reference test-suite with every
                      frozen order / verdict / witness of the hot path
  random_small.npz    seeded random graphs (n <= 90) with the reference's
                      LexBFS orders (LOWEST_INDEX, seeded array, parallel
                      ascending / descending / seeded) and is_peo results on
                      random permutations (verdict + witness)
  exhaustive5.npz     every labelled graph on n <= 5 vertices: order, verdict, witness
  configs.json        the BASELINE configurations: sha256 of the input
                      graphs, order fingerprints and witnesses (configs 1-5)
  configs_orders.npz  full LexBFS orders of configs 1 and 2 (int16)

Nothing in tests/ reads /root/reference at run time; the fixtures are the
reference's outputs frozen.
"""

from __future__ import annotations

import hashlib
import itertools
import json
import os
import random
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import chordalkit as C  # noqa: E402
from chordalkit.parallel import Arbitration, parallel_is_chordal, parallel_lexbfs  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def order0(o) -> list[int]:
    return [v - 1 for v in o]


def wit0(w):
    return None if w is None else [w.v - 1, w.p - 1, w.z - 1]


def named_graphs():
    sys.path.insert(0, "/root/reference/pkg/tests")
    import helpers as H

    return {
        "c4": H.c4(),
        "p3": H.p3(),
        "p3_relabeled": H.p3_relabeled(),
        "star5": H.star(5),
        "star8": H.star(8),
        "clique4": H.clique(4),
        "clique6": H.clique(6),
        "cycle7": H.cycle(7),
        "cycle9": H.cycle(9),
        "cycle16": H.cycle(16),
        "c5_chord_13": H.c5_chord_13(),
        "edgeless4": H.edgeless(4),
        "edgeless5": H.edgeless(5),
        "k1": C.Graph.from_edge_list(1, []),
        "k2": C.Graph.from_edge_list(2, [(1, 2)]),
        "disconnected6": C.Graph.from_edge_list(6, [(2, 5), (5, 6), (1, 3)]),
        "tree12_3": C.gen_tree(12, 3),
        "chordal14_3_5": C.gen_chordal_random(14, 3, 5),
        "chordal24_5_2": C.gen_chordal_random(24, 5, 2),
        "tree20_1": C.gen_tree(20, 1),
        "sparse150_5": C.gen_sparse_random(150, 5),
    }


def make_named():
    out = []
    for name, g in named_graphs().items():
        e = [[int(u), int(v)] for u, v in g.edges()]
        rec = {
            "name": name,
            "n": g.n,
            "edges": e,
            "lexbfs_partition": order0(C.lexbfs_partition(g)),
            "lexbfs_labels": order0(C.lexbfs_labels(g)),
            "par_asc": order0(parallel_lexbfs(g, Arbitration.fixed_priority())),
            "par_desc": order0(parallel_lexbfs(g, Arbitration.fixed_priority("descending"))),
            "par_seeded": {str(s): order0(parallel_lexbfs(g, Arbitration.seeded(s))) for s in (0, 3, 11)},
        }
        v = C.is_chordal(g)
        rec["chordal"] = v.chordal
        rec["witness"] = wit0(v.witness)
        pv = parallel_is_chordal(g, Arbitration.seeded(6))
        rec["par_seeded6_chordal"] = pv.chordal
        rec["par_seeded6_witness"] = wit0(pv.witness)
        out.append(rec)
    # frozen is_peo cases of test_peo.py / test_parallel_lexbfs.py
    H = named_graphs()
    peo_cases = []
    for gname, ordv in [
        ("c4", [1, 2, 4, 3]),
        ("clique4", [4, 2, 3, 1]),
        ("p3", [1, 2, 3]),
        ("star5", [1, 2, 3, 4, 5]),
        ("star5", [2, 3, 4, 5, 1]),
        ("cycle9", list(range(1, 10))),
    ]:
        ok, w = C.is_peo(H[gname], C.VertexOrdering(ordv))
        peo_cases.append({"graph": gname, "order": [v - 1 for v in ordv], "ok": ok, "witness": wit0(w)})
    with open(os.path.join(OUT, "named.json"), "w") as f:
        json.dump({"graphs": out, "peo_cases": peo_cases}, f, indent=0)


def make_random_small(count: int = 160):
    rng = random.Random(20261017)
    ns, packed, offs = [], [], [0]
    lex, desc, pseed, sarr, perms, pok, pw, cw = [], [], [], [], [], [], [], []
    for s in range(count):
        n = rng.choice([1, 2, 3, 5, 8, 13, 21, 31, 32, 33, 40, 47, 63, 64, 65, 77, 90])
        kind = s % 4
        if n < 3 or kind in (0, 1):
            p = (0.15, 0.3, 0.5, 0.7, 0.85)[s % 5]
            g = C.gen_dense_random(n, p, s) if n > 1 else C.Graph.from_edge_list(1, [])
        elif kind == 2:
            g = C.gen_chordal_random(n, min(n - 1, 1 + s % 6), s)
        else:
            g = C.gen_chordal_random(n, min(n - 1, 1 + s % 6), s)
            if n > 4:
                from paper_1508_06329_b200.generate import remove_first_chord  # noqa: E402

                g2, _ = remove_first_chord(C.Graph(g.n, g._packed.copy(), g.m))
                g = C.Graph(g2.n, np.array(g2._packed), g2.m)
        ns.append(n)
        packed.append(np.asarray(g._packed).reshape(-1))
        offs.append(offs[-1] + g._packed.size)
        lex.append(order0(C.lexbfs_partition(g)))
        desc.append(order0(parallel_lexbfs(g, Arbitration.fixed_priority("descending"))))
        pseed.append(order0(parallel_lexbfs(g, Arbitration.seeded(s))))
        sarr.append(order0(C.lexbfs_partition(g, C.seeded(s), method="array")))
        perm = list(range(1, n + 1))
        rng.shuffle(perm)
        perms.append([v - 1 for v in perm])
        ok, w = C.is_peo(g, C.VertexOrdering(perm))
        pok.append(ok)
        pw.append(wit0(w) or [-1, -1, -1])
        v = C.is_chordal(g)
        cw.append(wit0(v.witness) or [-1, -1, -1])
    flat = lambda xs: np.array([x for row in xs for x in row], dtype=np.int32)  # noqa: E731
    np.savez_compressed(
        os.path.join(OUT, "random_small.npz"),
        n=np.array(ns, dtype=np.int32),
        packed=np.concatenate(packed).astype(np.uint8),
        packed_off=np.array(offs, dtype=np.int64),
        lex=flat(lex),
        par_desc=flat(desc),
        par_seeded=flat(pseed),
        seeded_array=flat(sarr),
        perm=flat(perms),
        perm_ok=np.array(pok, dtype=bool),
        perm_witness=np.array(pw, dtype=np.int32),
        chordal_witness=np.array(cw, dtype=np.int32),
    )


def all_graphs(n):
    pairs = list(itertools.combinations(range(1, n + 1), 2))
    for mask in range(1 << len(pairs)):
        yield mask, C.Graph.from_edge_list(n, [p for i, p in enumerate(pairs) if mask >> i & 1])


def make_exhaustive5():
    ns, masks, orders, wits, chord = [], [], [], [], []
    for n in range(1, 6):
        for mask, g in all_graphs(n):
            ns.append(n)
            masks.append(mask)
            o = order0(C.lexbfs_partition(g))
            orders.append(o + [-1] * (5 - n))
            v = C.is_chordal(g)
            chord.append(v.chordal)
            wits.append(wit0(v.witness) or [-1, -1, -1])
    np.savez_compressed(
        os.path.join(OUT, "exhaustive5.npz"),
        n=np.array(ns, dtype=np.int8),
        mask=np.array(masks, dtype=np.int32),
        order=np.array(orders, dtype=np.int8),
        chordal=np.array(chord, dtype=bool),
        witness=np.array(wits, dtype=np.int8),
    )


def _record(g, label, t_lex=True):
    t0 = time.perf_counter()
    o = C.lexbfs_partition(g)
    t1 = time.perf_counter()
    ok, w = C.is_peo(g, o)
    t2 = time.perf_counter()
    o0 = np.asarray(o.order0, dtype=np.int32)
    print(f"  {label}: n={g.n} m={g.m} lexbfs {t1 - t0:.2f}s is_peo {t2 - t1:.2f}s chordal={ok} w={wit0(w)}",
          flush=True)
    return {
        "n": g.n,
        "m": int(g.m),
        "packed_sha256": sha(np.asarray(g._packed)),
        "order_sha256": sha(o0),
        "order_head": o0[:16].tolist(),
        "chordal": bool(ok),
        "witness": wit0(w),
        "ref_seconds": {"lexbfs_partition": t1 - t0, "is_peo": t2 - t1},
    }, o0


def _chord_removed(g):
    from paper_1508_06329_b200.generate import remove_first_chord  # noqa: E402

    h, e = remove_first_chord(g)
    return C.Graph(h.n, np.array(h._packed), h.m), e


def make_configs(which=("1", "2", "3", "4", "5")):
    path = os.path.join(OUT, "configs.json")
    res = json.load(open(path)) if os.path.exists(path) else {}
    opath = os.path.join(OUT, "configs_orders.npz")
    orders = dict(np.load(opath)) if os.path.exists(opath) else {}
    if "1" in which:
        print("config 1", flush=True)
        g = C.gen_chordal_random(1000, 8, 0)
        a, oa = _record(g, "chordal1000")
        h, e = _chord_removed(g)
        b, ob = _record(h, "chordal1000-chord")
        b["removed_edge"] = list(e)
        res["1"] = {"chordal": a, "nonchordal": b}
        orders["c1_chordal"], orders["c1_nonchordal"] = oa.astype(np.int16), ob.astype(np.int16)
    if "2" in which:
        print("config 2", flush=True)
        g = C.gen_dense_random(8192, 0.5, 0)
        a, oa = _record(g, "dense8192")
        g2 = C.gen_chordal_random(8192, 8, 0)
        b, ob = _record(g2, "chordal8192")
        res["2"] = {"dense": a, "chordal": b}
        orders["c2_dense"], orders["c2_chordal"] = oa.astype(np.int16), ob.astype(np.int16)
    if "3" in which:
        print("config 3", flush=True)
        g = C.gen_chordal_random(32768, 1024, 0, cap=32768)
        a, _ = _record(g, "chordal32768")
        h, e = _chord_removed(g)
        b, _ = _record(h, "chordal32768-chord")
        b["removed_edge"] = list(e)
        d = C.gen_dense_random(32768, 0.5, 0, cap=32768)
        c, _ = _record(d, "dense32768")
        res["3"] = {"chordal": a, "nonchordal": b, "dense": c}
    if "4" in which:
        print("config 4 sample", flush=True)
        sample = []
        for s in range(64):
            g = C.gen_dense_random(512, 0.5, s) if s % 2 == 0 else C.gen_chordal_random(512, 8, s)
            v = C.is_chordal(g)
            o0 = np.asarray(C.lexbfs_partition(g).order0, dtype=np.int32)
            sample.append({"seed": s, "packed_sha256": sha(np.asarray(g._packed)), "order_sha256": sha(o0),
                           "chordal": v.chordal, "witness": wit0(v.witness)})
        res["4"] = {"n": 512, "rule": "seed even: gen_dense_random(512,0.5,s); odd: gen_chordal_random(512,8,s)",
                    "sample": sample}
    if "5" in which:
        print("config 5", flush=True)
        res["5"] = make_config5()
    with open(path, "w") as f:
        json.dump(res, f, indent=1)
    np.savez_compressed(opath, **orders)


class _CSRShim:
    """Duck-typed graph exposing what the reference's linked LexBFS and list
    PEO read (n, m, adjacency_lists0) -- SURVEY §8(c)."""

    def __init__(self, n, indptr, indices):
        self.n = n
        self.m = int(indptr[-1]) // 2
        self._ip, self._ix = indptr, indices
        self._lists = None

    def adjacency_lists0(self):
        if self._lists is None:
            ip, ix = self._ip, self._ix
            self._lists = [ix[ip[v]:ip[v + 1]].tolist() for v in range(self.n)]
        return self._lists


def csr_from_edges(n, u, v):
    a = np.concatenate([u, v])
    b = np.concatenate([v, u])
    key = np.unique(a * n + b)
    rows, cols = key // n, key % n
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=indptr[1:])
    return indptr, cols.astype(np.int32)


def make_config5(n=1_000_000, k=8, seed=0):
    from paper_1508_06329_b200.generate import chordal_random_edges  # noqa: E402

    t0 = time.perf_counter()
    u, v = chordal_random_edges(n, k, seed)
    indptr, indices = csr_from_edges(n, u, v)
    t1 = time.perf_counter()
    shim = _CSRShim(n, indptr, indices)
    o = C.lexbfs_partition(shim, method="linked")
    t2 = time.perf_counter()
    ok, w = C.is_peo(shim, o, method="lists")
    t3 = time.perf_counter()
    o0 = np.asarray(o.order0, dtype=np.int32)
    print(f"  csr n={n} m={shim.m} gen {t1 - t0:.1f}s lexbfs {t2 - t1:.1f}s is_peo {t3 - t2:.1f}s ok={ok}", flush=True)
    # non-chordal twin: drop the first edge whose endpoints have two non-adjacent common neighbours
    lists = shim.adjacency_lists0()
    removed = None
    for a in range(n):
        for b in lists[a]:
            if b <= a:
                continue
            common = sorted(set(lists[a]) & set(lists[b]))
            bad = any(y not in set(lists[x]) for x, y in itertools.combinations(common, 2))
            if bad:
                removed = (a, b)
                break
        if removed:
            break
    keep = ~(((u == removed[1]) & (v == removed[0])) | ((u == removed[0]) & (v == removed[1])))
    ip2, ix2 = csr_from_edges(n, u[keep], v[keep])
    shim2 = _CSRShim(n, ip2, ix2)
    o2 = C.lexbfs_partition(shim2, method="linked")
    ok2, w2 = C.is_peo(shim2, o2, method="lists")
    o20 = np.asarray(o2.order0, dtype=np.int32)
    print(f"  csr nonchordal removed={removed} ok={ok2} w={wit0(w2)}", flush=True)
    return {
        "n": n, "k": k, "seed": seed, "m": shim.m,
        "indptr_sha256": sha(indptr), "indices_sha256": sha(indices),
        "order_sha256": sha(o0), "order_head": o0[:16].tolist(), "chordal": bool(ok), "witness": wit0(w),
        "ref_seconds": {"generate": t1 - t0, "lexbfs_partition_linked": t2 - t1, "is_peo_lists": t3 - t2},
        "nonchordal": {"removed_edge0": list(map(int, removed)), "order_sha256": sha(o20),
                       "chordal": bool(ok2), "witness": wit0(w2)},
    }


if __name__ == "__main__":
    sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
    what = sys.argv[1] if len(sys.argv) > 1 else "small"
    if what in ("small", "all"):
        make_named()
        make_random_small()
        make_exhaustive5()
        print("small fixtures written")
    if what in ("configs", "all"):
        make_configs(tuple(sys.argv[2].split(",")) if len(sys.argv) > 2 else ("1", "2", "3", "4", "5"))
