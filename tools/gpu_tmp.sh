bash tools/ab_variants.sh run "c5" labase la16e2 la32e2 la48e4 > gpurun_out/r02_ab_la2.txt 2>&1
grep -E "^(==|c)|Error" gpurun_out/r02_ab_la2.txt
