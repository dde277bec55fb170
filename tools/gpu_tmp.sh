bash tools/gpu_round.sh r02_v6
