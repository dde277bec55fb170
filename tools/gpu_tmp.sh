bash tools/ab_variants.sh run "batch c1" hbase hoff > gpurun_out/r02_ab_hoff.txt 2>&1
grep -E "^(==|c|b)|Error" gpurun_out/r02_ab_hoff.txt
