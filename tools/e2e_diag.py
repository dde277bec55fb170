"""Where the host-buffer batch call spends its time (pinned H2D, kernel, D2H, allocation).

    python tools/e2e_diag.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1508_06329_b200 import _native, ops  # noqa: E402


def main():
    B = 65536
    adj = bench.build_batch(0, B, "cuda")
    torch.cuda.synchronize()
    host = torch.empty(adj.shape, dtype=torch.uint8, pin_memory=True)
    host.copy_(adj)
    orders_h = torch.empty((B, 512), dtype=torch.int32, pin_memory=True)
    wit_h = torch.empty((B, 3), dtype=torch.int32, pin_memory=True)
    dev = torch.empty_like(adj)
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev.copy_(host, non_blocking=True)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        ops.is_chordal_batch(dev, 512, 64)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        for chunk in (4096, 8192, 16384):
            t3 = time.perf_counter()
            rc = _native.lib.chordal_is_chordal_batch_host(host.data_ptr(), B, 512, 64, orders_h.data_ptr(),
                                                           wit_h.data_ptr(), chunk)
            t4 = time.perf_counter()
            print(f"rep {rep} chunk {chunk}: host-API {1e3 * (t4 - t3):.1f} ms", flush=True)
        print(f"rep {rep}: H2D 2 GiB {1e3 * (t1 - t0):.1f} ms ({2.147 / (t1 - t0):.1f} GB/s), "
              f"kernel {1e3 * (t2 - t1):.1f} ms", flush=True)


if __name__ == "__main__":
    main()
