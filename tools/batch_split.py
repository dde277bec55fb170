"""Batch-kernel time split by graph family (config 4): all, dense-only, chordal-only.

    python tools/batch_split.py [graphs]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1508_06329_b200 import ops  # noqa: E402

import bench  # noqa: E402


def timeit(adj, reps=5):
    ops.is_chordal_batch(adj, 512, 64)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        ops.is_chordal_batch(adj, 512, 64)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    G = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    adj = bench.build_batch(0, G, "cuda")
    dense = adj[0::2].contiguous()
    chord = adj[1::2].contiguous()
    for name, x in (("all", adj), ("dense", dense), ("chordal", chord)):
        ms = timeit(x)
        print(f"{name:8s} graphs={x.shape[0]:6d} {ms:8.3f} ms  {x.shape[0] / ms * 1e3 / 1e6:7.3f} M graphs/s  "
              f"{ms * 1e6 / x.shape[0]:8.1f} ns/graph")


if __name__ == "__main__":
    main()
