set -x
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r02_v3_pytest_gpu.txt
cat gpurun_out/r02_v3_pytest_gpu.txt
bash tools/ab_variants.sh run "c5" ow_noef ow > gpurun_out/r02_ab_ef.txt 2>&1
L=paper_1508_06329_b200/lib/libchordal_b200.so
cp $L /tmp/keep.so; cp tools/exp/thr.so $L
for t in 64 128 256; do echo "== T=$t"; SEG_THREADS=$t timeout 300 python tools/variant_time.py c2c c3c; done > gpurun_out/r02_ab_threads.txt 2>&1
for t in 320 384; do echo "== T=$t"; SEG_THREADS=$t timeout 300 python tools/variant_time.py c3c c3r; done >> gpurun_out/r02_ab_threads.txt 2>&1
for t in 256 512 768 1024; do echo "== dense T=$t"; SEG_THREADS_DENSE=$t timeout 300 python tools/variant_time.py c2d c3d; done >> gpurun_out/r02_ab_threads.txt 2>&1
cp /tmp/keep.so $L
for t in racecheck memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_driver.py > gpurun_out/r02_v3_sanitize_${t}.txt 2>&1
  tail -2 gpurun_out/r02_v3_sanitize_${t}.txt
done
cat gpurun_out/r02_ab_ef.txt gpurun_out/r02_ab_threads.txt
