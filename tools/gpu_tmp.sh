bash tools/ab_variants.sh run "c5" laprev glob256 > gpurun_out/r02_ab_glob256.txt 2>&1
grep -E "^(==|c)|Error" gpurun_out/r02_ab_glob256.txt
