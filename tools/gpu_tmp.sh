set -x
bash tools/ab_variants.sh run "c3c c3r c3d c2c c2d" wt4 wt2 wt1 > gpurun_out/r02_ab_wt.txt 2>&1
grep -E "^(==|c)" gpurun_out/r02_ab_wt.txt
bash tools/ab_variants.sh run "c5" la32 laL1_8 laL1_16 > gpurun_out/r02_ab_laL1.txt 2>&1
grep -E "^(==|c)" gpurun_out/r02_ab_laL1.txt
