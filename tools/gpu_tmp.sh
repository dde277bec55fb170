bash tools/ab_variants.sh run "c3c c3r" sp_wt2 sp_mov128 sp_mov1k > gpurun_out/r02_ab_sparse3.txt 2>&1
grep -E "^(==|c)" gpurun_out/r02_ab_sparse3.txt
