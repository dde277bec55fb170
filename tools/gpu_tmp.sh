timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
bash tools/ab_variants.sh run "c3c c3r c3d c2c c2d" noeb4 eb4 > gpurun_out/r02_ab_eb4.txt 2>&1
grep -E "^(==|c)|Error" gpurun_out/r02_ab_eb4.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python tools/sanitize_driver.py cta > gpurun_out/r02_v10_sanitize_racecheck_cta.txt 2>&1
tail -2 gpurun_out/r02_v10_sanitize_racecheck_cta.txt
