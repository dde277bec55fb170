"""Host copy bandwidth with T threads over pinned buffers (sizing the e2e packer)."""
import os
import sys
import threading
import time

import numpy as np
import torch

n = 1 << 30
src = torch.empty(n, dtype=torch.uint8, pin_memory=True)
src.numpy()[:] = 1
dst = torch.empty(n // 2, dtype=torch.uint8, pin_memory=True)
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
for T in (1, 4, 8, 16, 32):
    a, b = src.numpy(), dst.numpy()
    per = n // T

    def work(t):
        s = a[t * per:(t + 1) * per]
        # copy the first half of every 64-byte row (the packer's access pattern)
        rows = s.reshape(-1, 64)
        d = b[t * per // 2:(t + 1) * per // 2].reshape(-1, 32)
        np.copyto(d, rows[:, 32:])

    ths = [threading.Thread(target=work, args=(t,)) for t in range(T)]
    t0 = time.perf_counter()
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    dt = time.perf_counter() - t0
    print(f"T={T:2d} read {n / dt / 1e9:6.1f} GB/s")
