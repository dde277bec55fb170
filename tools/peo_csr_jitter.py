"""Per-call times of the CSR PEO check on the config-5 graph (N = 10^6), to
separate kernel time from call-to-call variation.

    python tools/peo_csr_jitter.py [reps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1508_06329_b200 import ops  # noqa: E402
from paper_1508_06329_b200.generate import gen_chordal_random_csr_device  # noqa: E402


def timed(fn):
    """(device ms between events around the call, host ms spent inside the call)"""
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    t0 = time.perf_counter()
    fn()
    t1 = time.perf_counter()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e), (t1 - t0) * 1e3


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    n = 1_000_000
    ip, ix = gen_chordal_random_csr_device(n, 8, 0)
    o, p, par = ops.lexbfs_csr(ip, ix, n)
    torch.cuda.synchronize()
    for label, fn in (("peo_csr(parents)", lambda: ops.peo_csr(ip, ix, n, p, par)),
                      ("peo_csr(search)", lambda: ops.peo_csr(ip, ix, n, p)),
                      ("peo_csr_key(parents)", lambda: ops.peo_csr_key(ip, ix, n, p, 0, n, key, par))):
        key = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        ts = [timed(fn) for _ in range(reps)]
        print(label, "device", " ".join(f"{t[0]:.3f}" for t in ts))
        print(label, "host  ", " ".join(f"{t[1]:.3f}" for t in ts))
    # back to back, one event pair (what bench.py's time_events does)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        torch.cuda.synchronize()
        s.record()
        for _ in range(3):
            ops.peo_csr(ip, ix, n, p, par)
        e.record()
        torch.cuda.synchronize()
        print("3 back-to-back / 3", f"{s.elapsed_time(e) / 3:.3f}")


if __name__ == "__main__":
    main()
