# Final round evidence on one B200: smoke, GPU tests, bench (ours + reference arm), ncu launch list of the bench.
#   bash tools/gpu_final.sh TAG
TAG=${1:-r02_final}
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/${TAG}_pytest_gpu.txt
cat gpurun_out/${TAG}_pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2>gpurun_out/${TAG}_bench_ref.err
BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench_2rank_gloo.json 2> gpurun_out/${TAG}_bench_2rank_gloo.err
# (compute-sanitizer runs: the r02_final_sanitize_* logs; the tool is closed on this pool now)
[ -n "$NO_NCU" ] || timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/${TAG}_ncu_bench.log 2>&1
# the all-shared-memory CSR slot kernel on a CSR n = 8192 chordal graph (the 13th launch of c5_time.py)
[ -n "$NO_NCU" ] || timeout 900 ncu --set full --clock-control none --import-source on -k regex:lexbfs_csr_allsmem --launch-skip 12 -c 1 -o gpurun_out/${TAG}_slot8k python tools/c5_time.py > gpurun_out/${TAG}_ncu_slot8k.log 2>&1
ls -la gpurun_out
