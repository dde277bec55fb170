"""Time both LexBFS engines on the single-graph configurations (CUDA events).

    python tools/engine_compare.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1508_06329_b200 import _native, ops  # noqa: E402
from paper_1508_06329_b200.device import DeviceRows  # noqa: E402
from paper_1508_06329_b200.generate import chordal_random_edges, gen_dense_random_device  # noqa: E402
from paper_1508_06329_b200.graph import device_stride  # noqa: E402


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    cases = []
    for n, k in ((1000, 8), (8192, 8), (32768, 1024), (32768, 64), (32768, 8)):
        u, v = chordal_random_edges(n, k, 0)
        rows = DeviceRows(n, device_stride(n), ops.edges_to_dense(u, v, n, device_stride(n)))
        cases.append((f"chordal n={n} k={k}", rows))
    cases.append(("dense n=8192 p=.5", DeviceRows(8192, 1024, gen_dense_random_device(8192, 0.5, 0)[0])))
    cases.append(("dense n=32768 p=.5", DeviceRows(32768, 4096, gen_dense_random_device(32768, 0.5, 0)[0])))
    for name, rows in cases:
        m = ops.count_edges(rows)
        ip, ix = ops.dense_to_csr(rows)
        slot = t(lambda: ops.lexbfs_csr(ip, ix, rows.n))
        seg = t(lambda: ops.lexbfs(rows))  # n <= 32768: touched-segment arrangement engine
        o1, _, p1 = ops.lexbfs_csr(ip, ix, rows.n)
        o2, _, p2 = ops.lexbfs(rows, want_parent=True)
        same = bool(torch.equal(o1, o2))
        known = p2 != -2
        same_par = bool(torch.equal(p1[known], p2[known]))
        print(f"{name:24s} m={m:9d} avgdeg={2 * m / rows.n:7.1f}  slot(CSR) {slot:9.3f} ms "
              f"({slot * 1e6 / rows.n:8.1f} ns/step)  seg {seg:9.3f} ms ({seg * 1e6 / rows.n:8.1f} ns/step) "
              f"same_order={same} same_parent={same_par}", flush=True)


if __name__ == "__main__":
    main()
