bash tools/gpu_round.sh ${1:-r02k}
bash tools/profile_r02.sh ${1:-r02k}
