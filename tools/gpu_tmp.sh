bash tools/ab_variants.sh run "c3c c3r c3d c2c c2d" noagg aggf > gpurun_out/r02_ab_aggf.txt 2>&1
grep -E "^(==|c)|Error" gpurun_out/r02_ab_aggf.txt
