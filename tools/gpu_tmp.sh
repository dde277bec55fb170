bash tools/ab_variants.sh run "batch c1" hposbase bopt > gpurun_out/r02_ab_bopt.txt 2>&1
grep -E "^(==|c|b)|Error" gpurun_out/r02_ab_bopt.txt
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
