set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r01_pytest_gpu.txt
cat gpurun_out/r01_pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/r01_bench.json 2> gpurun_out/r01_bench.err
tail -3 gpurun_out/r01_bench.err
cat gpurun_out/r01_bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01_bench_ref.json 2>gpurun_out/r01_bench_ref.err
cat gpurun_out/r01_bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r01_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:batch -c 1 -o gpurun_out/r01_batch_full python tools/profile_driver.py batch > gpurun_out/r01_ncu_full.log 2>&1
ls -la gpurun_out
