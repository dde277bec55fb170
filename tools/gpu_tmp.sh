timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
bash tools/ab_variants.sh run "c1 c3c c3r" cur spoll > gpurun_out/r02_ab_spoll.txt 2>&1
grep -E "^(==|c)|Error" gpurun_out/r02_ab_spoll.txt
