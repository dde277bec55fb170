"""Write a chordal config graph as (int64 n, int64 stride, packed rows) for tools/seg_profile.

    python tools/dump_graph.py N K out.bin       (gen_chordal_random(N, K, 0))
    python tools/dump_graph.py N 0.5 out.bin     (gen_dense_random(N, 0.5, 0): a float second argument)
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1508_06329_b200.generate import chordal_random_edges  # noqa: E402
from paper_1508_06329_b200.graph import device_stride  # noqa: E402


def main(n, k, out):
    stride = device_stride(n)
    rows = np.zeros((n, stride), np.uint8)
    if "." in k:
        from paper_1508_06329_b200.generate import gen_dense_random

        g = gen_dense_random(n, float(k), 0, cap=max(n, 20000))
        rows[:, : g._packed.shape[1]] = g._packed
    else:
        u, v = chordal_random_edges(n, int(k), 0)
        for a, b in ((u, v), (v, u)):
            np.bitwise_or.at(rows, (a, b >> 3), (1 << (b & 7)).astype(np.uint8))
    with open(out, "wb") as f:
        np.array([n, stride], np.int64).tofile(f)
        rows.tofile(f)


def main_removed(n, k, out):
    """The chord-removed twin (generate.remove_first_chord) of gen_chordal_random(n, k, 0)."""
    from paper_1508_06329_b200.generate import gen_chordal_random, remove_first_chord

    g, _ = remove_first_chord(gen_chordal_random(n, int(k), 0, cap=max(n, 20000)))
    stride = device_stride(n)
    rows = np.zeros((n, stride), np.uint8)
    rows[:, : g._packed.shape[1]] = g._packed
    with open(out, "wb") as f:
        np.array([n, stride], np.int64).tofile(f)
        rows.tofile(f)


if __name__ == "__main__":
    if len(sys.argv) > 4 and sys.argv[4] == "x":
        main_removed(int(sys.argv[1]), sys.argv[2], sys.argv[3])
    else:
        main(int(sys.argv[1]), sys.argv[2], sys.argv[3])
