"""Small driver for ncu captures: runs each hot kernel a few times on config inputs.

    python tools/profile_driver.py {batch|batch_chordal|batch_dense|lexbfs32k|peo32k|lexbfs1k|csr1m|peo_csr1m|all}
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1508_06329_b200 import ops  # noqa: E402
from paper_1508_06329_b200.device import DeviceRows  # noqa: E402
from paper_1508_06329_b200.generate import chordal_random_edges  # noqa: E402

import bench  # noqa: E402


def rows_chordal(n, k, seed):
    u, v = chordal_random_edges(n, k, seed)
    stride = max(16, ((n + 7) // 8 + 15) // 16 * 16)
    return DeviceRows(n, stride, ops.edges_to_dense(u, v, n, stride))


def main(what):
    if what in ("batch", "all", "batch_chordal", "batch_dense"):
        adj = bench.build_batch(0, int(os.environ.get("GRAPHS", "16384")), "cuda")
        if what == "batch_chordal":
            adj = adj[1::2].contiguous()
        elif what == "batch_dense":
            adj = adj[0::2].contiguous()
        for _ in range(3):
            ops.is_chordal_batch(adj, 512, 64)
    if what in ("lexbfs32k", "peo32k", "all"):
        r = rows_chordal(32768, 1024, 0)
        for _ in range(2):
            order, pos, parent = ops.lexbfs(r, want_parent=True)
            ops.peo(r, order, pos, parent)  # the pipeline form (parents from LexBFS)
            ops.peo(r, order, pos)          # standalone is_peo (parents searched)
    if what == "lexbfs8k":
        r = rows_chordal(8192, 8, 0)
        ops.lexbfs(r)
    if what == "csr1m":
        from paper_1508_06329_b200.generate import gen_chordal_random_csr_device

        ip, ix = gen_chordal_random_csr_device(1_000_000, 8, 0)
        ops.lexbfs_csr(ip, ix, 1_000_000)
    if what == "peo_csr1m":
        from paper_1508_06329_b200.generate import gen_chordal_random_csr_device

        ip, ix = gen_chordal_random_csr_device(1_000_000, 8, 0)
        order, pos, parent = ops.lexbfs_csr(ip, ix, 1_000_000)
        ws = ops.peo_csr_workspace(1_000_000, ip.device)
        for _ in range(3):
            ops.peo_csr(ip, ix, 1_000_000, pos, parent, ws=ws)
    if what in ("lexbfs1k", "all"):
        r = rows_chordal(1000, 8, 0)
        for _ in range(3):
            ops.is_chordal(r)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
