"""Time the LexBFS engines on one dense-stored graph: touched-segment CTA kernel
(ops.lexbfs) vs the CSR slot engine on a device-built CSR (ops.lexbfs_csr).

    python tools/engine_time.py N K      (gen_chordal_random(N, K, 0))
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


def main(n, k):
    u, v = chordal_random_edges(n, k, 0)
    rows = DeviceRows(n, device_stride(n), ops.edges_to_dense(u, v, n, device_stride(n)), m=len(u))
    ip, ix = ops.csr_from_rows(rows)
    seg = bench.time_events(lambda: ops.lexbfs(rows))
    slot = bench.time_events(lambda: ops.lexbfs_csr(ip, ix, n, m=len(u)))
    a = ops.lexbfs(rows)[0].cpu()
    b = ops.lexbfs_csr(ip, ix, n, m=len(u))[0].cpu()
    print(f"n={n} k={k} m={len(u)} seg {seg:.3f} ms ({seg * 1e6 / n:.0f} ns/step)  "
          f"slot {slot:.3f} ms ({slot * 1e6 / n:.0f} ns/step)  same={torch.equal(a, b)}")


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]))
