"""Where does the CSR slot engine (all state in shared memory) beat the touched-segment
CTA engine on dense-stored sparse graphs?  Times both LexBFS engines (CUDA events)
on gen_chordal_random(n, k, 0) for a grid of n and k.

    python tools/engine_cross.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1508_06329_b200 import ops  # noqa: E402
from paper_1508_06329_b200.device import DeviceRows  # noqa: E402
from paper_1508_06329_b200.generate import chordal_random_edges  # noqa: E402
from paper_1508_06329_b200.graph import device_stride  # noqa: E402

import bench  # noqa: E402


def main():
    for n in (1500, 2048, 4096, 8192):
        for k in (4, 8, 16, 32):
            u, v = chordal_random_edges(n, k, 0)
            rows = DeviceRows(n, device_stride(n), ops.edges_to_dense(u, v, n, device_stride(n)), m=len(u))
            ip, ix = ops.dense_to_csr(rows)
            seg = bench.time_events(lambda: ops.lexbfs(rows), reps=5)
            slot = bench.time_events(lambda: ops.lexbfs_csr(ip, ix, n, m=len(u)), reps=5)
            conv = bench.time_events(lambda: ops.dense_to_csr(rows), reps=5)
            same = torch.equal(ops.lexbfs(rows)[0], ops.lexbfs_csr(ip, ix, n, m=len(u))[0])
            print(f"n={n:5d} k={k:2d} avgdeg={2 * len(u) / n:6.1f} seg {seg:7.3f} ms  slot {slot:7.3f} ms  "
                  f"(+csr conversion {conv:6.3f} ms)  slot/seg {slot / seg:5.2f} same={same}", flush=True)


if __name__ == "__main__":
    main()
