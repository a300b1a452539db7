bash tools/gpu_round.sh r02k
bash tools/profile_r02.sh r02k
