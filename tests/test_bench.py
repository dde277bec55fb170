"""bench.py on CPU: the reference arm, the oracle's generators it draws from, and
the multi-rank protocol of the main arm (torchrun, gloo, world_size 2).

The reference arm must never load the product library (its timed loop is the
oracle's C port of the reference, on the reference generators' graphs), must
name the same configuration as the GPU arm, and under torchrun only rank 0
prints.
"""

import hashlib
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, load_json

import oracle


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_oracle_generators_match_reference_config4_sample():
    cfg = load_json("configs.json")["4"]
    for rec in cfg["sample"]:
        s = rec["seed"]
        g = oracle.gen_dense_random(512, 0.5, s) if s % 2 == 0 else oracle.gen_chordal_random(512, 8, s)
        assert _sha(g) == rec["packed_sha256"], s


def test_oracle_batch_generator_matches_single_generators():
    b = oracle.gen_config4_batch(37, 12, nthreads=3)
    for i in range(12):
        s = 37 + i
        g = oracle.gen_dense_random(512, 0.5, s, 64) if s % 2 == 0 else oracle.gen_chordal_random(512, 8, s, 64)
        assert np.array_equal(b[i], g)


@pytest.mark.parametrize("which", ["1-chordal", "2-chordal", "2-dense"])
def test_oracle_generators_match_reference_configs(which):
    cfg, kind = which.split("-")
    rec = load_json("configs.json")[cfg][kind]
    n = rec["n"]
    g = oracle.gen_chordal_random(n, 8, 0) if kind == "chordal" else oracle.gen_dense_random(n, 0.5, 0)
    assert _sha(g) == rec["packed_sha256"]


def _run_bench(args, env_extra=None, torchrun=0):
    env = dict(os.environ, PYTHONPATH=ROOT)
    env.pop("CUDA_VISIBLE_DEVICES", None)
    env.update(env_extra or {})
    # record which shared objects the process mapped, and whether the product
    # package was imported, from inside the bench process itself
    probe = (
        "import atexit, sys, runpy\n"
        "def _report():\n"
        "    maps = open('/proc/self/maps').read()\n"
        "    sys.stderr.write('PROBE ' + repr(('libchordal_b200' in maps, 'paper_1508_06329_b200' in sys.modules))"
        " + '\\n')\n"
        "atexit.register(_report)\n"
        f"sys.argv = ['bench.py'] + {args!r}\n"
        f"runpy.run_path({os.path.join(ROOT, 'bench.py')!r}, run_name='__main__')\n"
    )
    if torchrun:
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        path = os.path.join(ROOT, "gpurun_out", "_bench_probe.py")
        os.makedirs(os.path.dirname(path), exist_ok=True)
        with open(path, "w") as f:
            f.write(probe)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={torchrun}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", path]
    else:
        cmd = [sys.executable, "-c", probe]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return r


def _json_lines(text):
    return [json.loads(x) for x in text.splitlines() if x.startswith("{")]


def test_reference_arm_never_loads_the_product():
    r = _run_bench(["--impl", "reference", "--graphs", "256", "--steps", "1", "--warmup", "1"])
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    line = lines[0]
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "config", "cpu_baseline", "e2e", "impl"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["value"] == line["value"] and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["value"] == line["value"]
    assert "PROBE (False, False)" in r.stderr  # no libchordal_b200.so mapped, package never imported
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    assert line["config"] == bench.config4(256)  # the GPU arm names the identical dict
    assert line["chordal_fraction"] == 0.5  # odd seeds are the chordal family


def test_reference_arm_under_torchrun_prints_once():
    r = _run_bench(["--impl", "reference", "--graphs", "128", "--steps", "1", "--warmup", "0"], torchrun=2)
    lines = _json_lines(r.stdout)
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2
    assert r.stderr.count("PROBE (False, False)") == 2


def test_shard_tiles_exactly():
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    for total in (1, 7, 65536, 65537, 99999):
        for world in (1, 2, 3, 4, 5, 6, 7, 8):
            parts = [bench.shard(total, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))


_DIST_WORKER = r'''
import json, os, sys
import numpy as np
import torch.distributed as dist
sys.path.insert(0, os.environ["BENCH_ROOT"])
import importlib.util
spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(os.environ["BENCH_ROOT"], "bench.py"))
bench = importlib.util.module_from_spec(spec); spec.loader.exec_module(bench)
import oracle
rank, world, _ = bench.dist_env()
dist.init_process_group("gloo")
G = 96
lo, hi = bench.shard(G, rank, world)
adj = oracle.gen_config4_batch(lo, hi - lo, nthreads=2)
verdict, orders, wit = oracle.is_chordal_batch(adj, 512, nthreads=2)
chordal, graphs = bench.reduce_sum_ints([int(verdict.sum()), hi - lo], world)
t = bench.reduce_max(float(rank + 1), world)
bench.barrier(world)
if rank == 0:
    print(json.dumps({"chordal": chordal, "graphs": graphs, "tmax": t, "world": world}))
dist.destroy_process_group()
'''


def test_multi_rank_protocol_gloo_world2():
    """The main arm's rank plumbing (exact shards, SUM of per-rank verdict counts,
    MAX of per-rank times, barrier) on two gloo ranks, per-rank work from the oracle."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    path = os.path.join(ROOT, "gpurun_out", "_bench_dist_worker.py")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as f:
        f.write(_DIST_WORKER)
    env = dict(os.environ, BENCH_ROOT=ROOT, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", f"--master-port={port}", path],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    out = _json_lines(r.stdout)
    assert len(out) == 1
    assert out[0] == {"chordal": 48, "graphs": 96, "tmax": 2.0, "world": 2}
