bash tools/ab_variants.sh run "batch c1" bopt bopt3 > gpurun_out/r02_ab_bopt3.txt 2>&1
grep -E "^(==|c|b)|Error" gpurun_out/r02_ab_bopt3.txt
