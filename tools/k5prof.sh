timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_energy_fid -c 1 -o gpurun_out/k5_cur -f python tools/solver_probe.py > /dev/null 2>&1
ncu -i gpurun_out/k5_cur.ncu-rep --page raw --csv > gpurun_out/k5_cur.raw.csv 2>/dev/null
rm -f gpurun_out/k5_cur.ncu-rep
