set -x
bash tools/gpu_final.sh r02_final4
