"""Where do the occasional slow host-buffer batch calls come from?  Times 12 calls of
(a) chordal_is_chordal_batch_host and (b) the same pipeline driven from Python with
persistent device buffers and streams (H2D chunk -> batch kernel -> D2H on 3 streams)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1508_06329_b200 import _native  # noqa: E402

import bench  # noqa: E402

B, N, S, CH = 65536, 512, 64, 8192
adj = bench.build_batch(0, B, "cuda")
host = torch.empty((B, N, S), dtype=torch.uint8, pin_memory=True)
host.copy_(adj)
orders_h = torch.empty((B, N), dtype=torch.int32, pin_memory=True)
wit_h = torch.empty((B, 3), dtype=torch.int32, pin_memory=True)
lib = _native.lib


def api():
    rc = lib.chordal_is_chordal_batch_host(host.data_ptr(), B, N, S, orders_h.data_ptr(), wit_h.data_ptr(), CH)
    assert rc == 0


streams = [torch.cuda.Stream() for _ in range(3)]
bufs = [torch.empty((CH, N, S), dtype=torch.uint8, device="cuda") for _ in range(3)]
ords = [torch.empty((CH, N), dtype=torch.int32, device="cuda") for _ in range(3)]
wits = [torch.empty((CH, 3), dtype=torch.int32, device="cuda") for _ in range(3)]


def manual():
    for c, b0 in enumerate(range(0, B, CH)):
        k = c % 3
        with torch.cuda.stream(streams[k]):
            bufs[k].copy_(host[b0:b0 + CH], non_blocking=True)
            rc = lib.chordal_is_chordal_batch(bufs[k].data_ptr(), CH, N, S, ords[k].data_ptr(), wits[k].data_ptr(),
                                              streams[k].cuda_stream)
            assert rc == 0
            orders_h[b0:b0 + CH].copy_(ords[k], non_blocking=True)
            wit_h[b0:b0 + CH].copy_(wits[k], non_blocking=True)
    torch.cuda.synchronize()


for name, fn in (("api", api), ("manual", manual), ("api", api)):
    for _ in range(3):
        fn()
    t = []
    for _ in range(12):
        t0 = time.perf_counter()
        fn()
        t.append(round(1e3 * (time.perf_counter() - t0), 1))
    print(name, t)
