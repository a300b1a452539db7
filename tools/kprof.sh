# usage: bash tools/kprof.sh <kernel-regex> <tag> <script> [env...]
# One ncu --set full capture of the first matching launch, exported to CSV in gpurun_out/.
k=$1; tag=$2; script=$3; shift 3
env "$@" timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
  -o gpurun_out/$tag -f python $script > /dev/null 2>&1
ncu -i gpurun_out/$tag.ncu-rep --page raw --csv > gpurun_out/$tag.raw.csv 2>/dev/null
ncu -i gpurun_out/$tag.ncu-rep --page source --csv > gpurun_out/$tag.src.csv 2>/dev/null
rm -f gpurun_out/$tag.ncu-rep
