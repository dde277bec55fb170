bash tools/ab_variants.sh run "batch" mb9 mb8 mb10 > gpurun_out/r02_ab_minb.txt 2>&1
grep -E "^(==|c|b)|Error" gpurun_out/r02_ab_minb.txt
