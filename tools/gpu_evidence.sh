# ncu --set full captures of the single-graph kernels + compute-sanitizer logs.
#   bash tools/gpu_evidence.sh TAG
TAG=${1:-r02}
set -x
for t in memcheck racecheck synccheck; do
  for part in warp cta slot peo other; do
    timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_driver.py $part \
      > gpurun_out/${TAG}_sanitize_${t}_${part}.txt 2>&1
    tail -3 gpurun_out/${TAG}_sanitize_${t}_${part}.txt
  done
done
[ -n "$NO_NCU" ] && exit 0
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lexbfs_seg -c 1 -o gpurun_out/${TAG}_seg32k python tools/profile_driver.py lexbfs32k > gpurun_out/${TAG}_ncu_seg32k.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:peo_csr -c 2 -o gpurun_out/${TAG}_peocsr1m python tools/profile_driver.py peo_csr1m > gpurun_out/${TAG}_ncu_peocsr.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:lexbfs_csr -c 1 -o gpurun_out/${TAG}_csr1m python tools/profile_driver.py csr1m > gpurun_out/${TAG}_ncu_csr1m.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:batch -c 1 -o gpurun_out/${TAG}_batch_full env GRAPHS=16384 python tools/profile_driver.py batch > gpurun_out/${TAG}_ncu_batch.log 2>&1
ls -la gpurun_out
