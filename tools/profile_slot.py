"""ncu driver: the CSR slot engine on configuration 3 (n = 32768, k = 1024)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1508_06329_b200 import ops  # noqa: E402
from paper_1508_06329_b200.device import DeviceRows  # noqa: E402
from paper_1508_06329_b200.generate import chordal_random_edges  # noqa: E402

n, k = int(os.environ.get("N", "32768")), int(os.environ.get("K", "1024"))
u, v = chordal_random_edges(n, k, 0)
stride = max(16, ((n + 7) // 8 + 15) // 16 * 16)
rows = DeviceRows(n, stride, ops.edges_to_dense(u, v, n, stride))
ip, ix = ops.dense_to_csr(rows)
ops.lexbfs_csr(ip, ix, n)
torch.cuda.synchronize()
