# Round-end evidence on one B200: GPU tests, bench (ours + reference arm),
# ncu launch list of the bench, ncu --set full of the batch kernel.
#   bash tools/gpu_round.sh TAG
TAG=${1:-r01}
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/${TAG}_pytest_gpu.txt
cat gpurun_out/${TAG}_pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -3 gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2>gpurun_out/${TAG}_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/${TAG}_ncu_bench.log 2>&1
GRAPHS=16384 timeout 900 ncu --set full --clock-control none --import-source on -k regex:batch -c 1 -o gpurun_out/${TAG}_batch_full python tools/profile_driver.py batch > gpurun_out/${TAG}_ncu_full.log 2>&1
ls -la gpurun_out
