"""Config-5 CSR PEO check timing (device, CUDA events) for the group sizes of
peo_csr_kernel, with and without the LexBFS parents, plus violating orders;
results checked against the oracle.  python tools/peo_csr_time.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_1508_06329_b200 import ops  # noqa: E402
from paper_1508_06329_b200.generate import gen_chordal_random_csr_device  # noqa: E402

n = 1_000_000
ip, ix = gen_chordal_random_csr_device(n, 8, 0)
t0 = time.perf_counter()
order, pos, par = ops.lexbfs_csr(ip, ix, n)
torch.cuda.synchronize()
print(f"lexbfs {time.perf_counter() - t0:.2f}s", flush=True)
ws = ops.peo_csr_workspace(n, ip.device)
ip_h, ix_h = ip.cpu().numpy(), ix.cpu().numpy()
o_h = order.cpu().numpy()
# a violating order: reverse a window in the middle
bad = o_h.copy()
bad[400000:400200] = bad[400000:400200][::-1].copy()
bad_d = torch.as_tensor(bad).cuda()
bad_pos = ops.positions(bad_d)
ok_b, w_b = oracle.is_peo_csr(ip_h, ix_h, n, bad)
print("oracle bad:", ok_b, w_b, flush=True)


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(20_000_000)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


deg = np.diff(ip_h)
for thr in (256, 1024, 4096, 65536, 1 << 30):
    print(f"rows with deg > {thr}: {(deg > thr).sum()}, entries {deg[deg > thr].sum()}", flush=True)
for g, thr in [(8, 256)]:
    a = timeit(lambda: ops.peo_csr(ip, ix, n, pos, par, ws=ws))
    b = timeit(lambda: ops.peo_csr(ip, ix, n, pos, None, ws=ws))
    c = timeit(lambda: ops.peo_csr(ip, ix, n, bad_pos, None, ws=ws))
    w1 = ops.witness_tuple(ops.peo_csr(ip, ix, n, pos, par, ws=ws))
    w2 = ops.witness_tuple(ops.peo_csr(ip, ix, n, pos, None, ws=ws))
    w3 = ops.witness_tuple(ops.peo_csr(ip, ix, n, bad_pos, None, ws=ws))
    print(f"G={g:2d} heavy>{thr}: parents given {a:.3f} ms  searched {b:.3f} ms  violating {c:.3f} ms  "
          f"ok={w1 is None and w2 is None} bad={w3 == w_b} {w3}", flush=True)
