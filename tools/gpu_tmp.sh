set -x
bash tools/ab_variants.sh run "c3c c3r c3d c2c c2d" base fp > gpurun_out/r02_ab_fp.txt 2>&1
grep -E "^(==|c)" gpurun_out/r02_ab_fp.txt
