"""Time the CSR slot engine on configuration 5 (gen_chordal_random(10^6, 8, 0), CSR)
and on smaller CSR graphs; prints a sha of each order so variants can be compared.

    python tools/c5_time.py
"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1508_06329_b200 import ops  # noqa: E402
from paper_1508_06329_b200.generate import gen_chordal_random_csr_device  # noqa: E402

import bench  # noqa: E402


def main():
    for n, k in ((1000, 8), (8192, 8), (16384, 8), (1000000, 8)):
        ip, ix = gen_chordal_random_csr_device(n, k, 0)
        m = int(ix.numel()) // 2
        t = bench.time_events(lambda: ops.lexbfs_csr(ip, ix, n, m=m), reps=3 if n > 100000 else 10)
        o = ops.lexbfs_csr(ip, ix, n, m=m)[0].cpu().numpy()
        print(f"csr n={n} k={k} m={m}: {t:.3f} ms ({t * 1e6 / n:.0f} ns/step) "
              f"sha {hashlib.sha256(o.tobytes()).hexdigest()[:16]}", flush=True)


if __name__ == "__main__":
    main()
