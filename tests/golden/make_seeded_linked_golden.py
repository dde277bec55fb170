"""Golden vectors for the seeded *linked* LexBFS variants: run the REFERENCE on
random graphs and freeze its orders.

    cd /tmp && PYTHONPATH=/root/reference/pkg/src python /root/repo/tests/golden/make_seeded_linked_golden.py

For every graph i (packed rows in the npz) and its seed s_i:
  part[i]   lexbfs_partition(g, seeded(s_i), method="linked")  (search.py:500-532)
  labels[i] lexbfs_labels(g, seeded(s_i), method="linked")     (search.py:262-310)
  chordal[i], witness[i]  is_chordal(g, "partition", seeded(s_i), method="reference")
  mcs[i], mcs_seeded[i], bfs[i], bfs_seeded[i]   mcs_order / bfs_order (search.py:79-145),
                          LOWEST_INDEX and seeded(s_i)
Orders are 0-based, padded with -1.
"""
import os
import random

import numpy as np
from chordalkit.generate import gen_chordal_random, gen_dense_random
from chordalkit.graph import Graph
from chordalkit.peo import is_chordal
from chordalkit.search import bfs_order, lexbfs_labels, lexbfs_partition, mcs_order, seeded

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "seeded_linked.npz")


def main():
    rng = random.Random(20151508)
    graphs = []
    for i in range(90):
        kind = i % 6
        n = rng.randint(1, 90)
        if kind == 0:
            g = gen_dense_random(n, rng.choice([0.05, 0.2, 0.5, 0.9]), i)
        elif kind in (1, 2):
            g = gen_chordal_random(n, rng.randint(0, max(0, min(6, n - 1))), i) if n > 1 else gen_dense_random(n, 0.5, i)
        elif kind == 3:  # disconnected: a few components
            edges = [(u, v) for u in range(1, n + 1) for v in range(u + 1, n + 1) if rng.random() < 0.04]
            g = Graph.from_edge_list(n, edges)
        elif kind == 4:  # cycles and paths
            edges = [(v, v % n + 1) for v in range(1, n + 1) if v % n + 1 != v and rng.random() < 0.9]
            g = Graph.from_edge_list(n, list({tuple(sorted(e)) for e in edges}))
        else:
            g = gen_dense_random(n, 0.3, 1000 + i)
        graphs.append(g)
    graphs.append(gen_chordal_random(1500, 8, 3))
    graphs.append(gen_dense_random(1100, 0.02, 4))
    N = max(g.n for g in graphs)
    W = (N + 7) // 8
    B = len(graphs)
    packed = np.zeros((B, N, W), np.uint8)
    ns = np.zeros(B, np.int64)
    seeds = np.zeros(B, np.int64)
    part = -np.ones((B, N), np.int32)
    labels = -np.ones((B, N), np.int32)
    chordal = np.zeros(B, np.bool_)
    witness = -np.ones((B, 3), np.int32)
    extra = {k: -np.ones((B, N), np.int32) for k in ("mcs", "mcs_seeded", "bfs", "bfs_seeded")}
    for i, g in enumerate(graphs):
        s = rng.randint(-5, 10**12)
        ns[i], seeds[i] = g.n, s
        packed[i, : g.n, : g._packed.shape[1]] = g._packed
        part[i, : g.n] = np.asarray(lexbfs_partition(g, seeded(s), method="linked").order) - 1
        labels[i, : g.n] = np.asarray(lexbfs_labels(g, seeded(s), method="linked").order) - 1
        if g.n <= 400:  # the reference's MCS is O(n^2) in Python
            extra["mcs"][i, : g.n] = np.asarray(mcs_order(g).order) - 1
            extra["mcs_seeded"][i, : g.n] = np.asarray(mcs_order(g, seeded(s)).order) - 1
        extra["bfs"][i, : g.n] = np.asarray(bfs_order(g).order) - 1
        extra["bfs_seeded"][i, : g.n] = np.asarray(bfs_order(g, seeded(s)).order) - 1
        v = is_chordal(g, "partition", seeded(s), method="reference")
        chordal[i] = v.chordal
        if not v.chordal:
            w = v.witness
            witness[i] = (w.v - 1, w.p - 1, w.z - 1)
    np.savez_compressed(OUT, packed=packed, n=ns, seed=seeds, part=part, labels=labels, chordal=chordal,
                        witness=witness, **extra)
    print(B, "graphs ->", OUT)


if __name__ == "__main__":
    main()
