"""Repeated pinned host->device copies of the config-4 batch size (2 GiB): are the
e2e outliers in our host API or in the box's copy path?"""
import time

import torch

n = 2 << 30
host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
host.fill_(1)
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
out = []
for i in range(15):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    out.append(round(1e3 * (time.perf_counter() - t0), 2))
print("2 GiB pinned H2D ms:", out)
