"""Time the hot kernels of the in-tree library on the config inputs (CUDA events).

    python tools/variant_time.py [c1 c2c c2d c3c c3r c3d c5 c5peo batch ...]

Used for A/B runs: build variants with CHORDAL_NVCC_EXTRA into copies of the
library, copy each into place in turn (tools/ab_variants.sh) and compare lines.
Each line also checks the order / verdict against the default build's result
hash written by the first run (same inputs, so every variant must agree).
"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1508_06329_b200 import ops  # noqa: E402
from paper_1508_06329_b200.device import DeviceRows  # noqa: E402
from paper_1508_06329_b200.generate import (  # noqa: E402
    chordal_random_edges,
    gen_chordal_random_csr_device,
    gen_dense_random_device,
)
from paper_1508_06329_b200.graph import device_stride  # noqa: E402

import bench  # noqa: E402

HASHES = os.environ.get("VARIANT_HASHES", "/tmp/variant_hashes.json")


def chordal_rows(n, k, seed=0, drop_first_chord=False):
    if drop_first_chord:
        from paper_1508_06329_b200.device import device_rows
        from paper_1508_06329_b200.generate import gen_chordal_random, remove_first_chord

        return device_rows(remove_first_chord(gen_chordal_random(n, k, seed, cap=n))[0])
    u, v = chordal_random_edges(n, k, seed)
    return DeviceRows(n, device_stride(n), ops.edges_to_dense(u, v, n, device_stride(n)), m=len(u))


def dense_rows(n, p, seed=0):
    st = device_stride(n)
    return DeviceRows(n, st, gen_dense_random_device(n, p, range(seed, seed + 1), stride=st)[0])


def h(t):
    return hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()[:12]


def run(name):
    if name in ("c1", "c2c", "c2d", "c3c", "c3r", "c3d"):
        rows = {
            "c1": lambda: chordal_rows(1000, 8),
            "c2c": lambda: chordal_rows(8192, 8),
            "c2d": lambda: dense_rows(8192, 0.5),
            "c3c": lambda: chordal_rows(32768, 1024),
            "c3r": lambda: chordal_rows(32768, 1024, drop_first_chord=True),
            "c3d": lambda: dense_rows(32768, 0.5),
        }[name]()
        reps = 3 if rows.n >= 32768 else 10
        ms = bench.time_events(lambda: ops.lexbfs(rows), reps=reps)
        tot = bench.time_events(lambda: ops.is_chordal(rows), reps=reps)
        order = ops.lexbfs(rows)[0]
        return {"lexbfs_ms": ms, "is_chordal_ms": tot, "ns_per_step": ms * 1e6 / rows.n, "hash": h(order)}
    if name in ("c5", "c5peo"):
        n = 1_000_000
        ip, ix = gen_chordal_random_csr_device(n, 8, 0)
        if name == "c5":
            ms = bench.time_events(lambda: ops.lexbfs_csr(ip, ix, n), reps=2)
            order = ops.lexbfs_csr(ip, ix, n)[0]
            return {"lexbfs_ms": ms, "ns_per_step": ms * 1e6 / n, "hash": h(order)}
        order, pos, parent = ops.lexbfs_csr(ip, ix, n)
        ws = ops.peo_csr_workspace(n, ip.device)
        ms = bench.time_events(lambda: ops.peo_csr(ip, ix, n, pos, parent, ws=ws), reps=20)
        ms2 = bench.time_events(lambda: ops.peo_csr(ip, ix, n, pos, None, ws=ws), reps=20)
        return {"peo_ms_parents": ms, "peo_ms_search": ms2}
    if name == "batch":
        adj = bench.build_batch(0, 65536, "cuda")
        ms = bench.time_events(lambda: ops.is_chordal_batch(adj, 512, 64), reps=5)
        out = ops.is_chordal_batch(adj, 512, 64)
        return {"batch_ms": ms, "graphs_per_s": 65536 / ms * 1e3, "hash": h(out[0])}
    raise SystemExit(f"unknown workload {name}")


def main(names):
    torch.cuda.set_device(0)
    known = json.load(open(HASHES)) if os.path.exists(HASHES) else {}
    for name in names:
        r = run(name)
        if "hash" in r:
            if name in known and known[name] != r["hash"]:
                r["MISMATCH"] = known[name]
            known.setdefault(name, r["hash"])
        print(name, json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
    json.dump(known, open(HASHES, "w"))


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2c", "c3c", "c5", "batch"])
