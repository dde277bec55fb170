set -x
bash tools/gpu_final.sh r02_final
TAG=r02_final
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lexbfs_seg -c 1 -o gpurun_out/${TAG}_seg32k python tools/profile_driver.py lexbfs32k > gpurun_out/${TAG}_ncu_seg32k.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lexbfs_seg -c 1 -o gpurun_out/${TAG}_seg8k python tools/profile_driver.py lexbfs8k > gpurun_out/${TAG}_ncu_seg8k.log 2>&1
GRAPHS=16384 timeout 900 ncu --set full --clock-control none --import-source on -k regex:batch -c 1 -o gpurun_out/${TAG}_batch_full python tools/profile_driver.py batch > gpurun_out/${TAG}_ncu_batch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:lexbfs_csr -c 1 -o gpurun_out/${TAG}_csr1m python tools/profile_driver.py csr1m > gpurun_out/${TAG}_ncu_csr1m.log 2>&1
ls -la gpurun_out
