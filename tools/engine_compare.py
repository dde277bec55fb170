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
    for name, rows in cases:
        m = ops.count_edges(rows)
        ip, ix = ops.dense_to_csr(rows)
        slot = t(lambda: ops.lexbfs_csr(ip, ix, rows.n))
        arr = t(lambda: ops.lexbfs(DeviceRows(rows.n, rows.stride, rows.data, 10**12)))  # force arrangement
        o1 = ops.lexbfs_csr(ip, ix, rows.n)[0]
        o2 = ops.lexbfs(DeviceRows(rows.n, rows.stride, rows.data, 10**12))[0]
        same = bool(torch.equal(o1, o2))
        print(f"{name:24s} m={m:9d} avgdeg={2 * m / rows.n:7.1f}  slot(smem/L2) {slot:9.3f} ms "
              f"({slot * 1e6 / rows.n:8.1f} ns/step)  arrangement {arr:9.3f} ms  same={same}", flush=True)


if __name__ == "__main__":
    main()
