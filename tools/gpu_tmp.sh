bash tools/ab_variants.sh run "c3c c3r c3d c2c c2d" mvbase mvd2 mvs1 > gpurun_out/r02_ab_mv.txt 2>&1
grep -E "^(==|c)|Error" gpurun_out/r02_ab_mv.txt
