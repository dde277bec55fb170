bash tools/ab_variants.sh run "c3c c3r" k1 k2 k4 > gpurun_out/r02_ab_spank.txt 2>&1
grep -E "^(==|c)|Error" gpurun_out/r02_ab_spank.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "oracle or config3 or config2" 2>&1 | tail -2
