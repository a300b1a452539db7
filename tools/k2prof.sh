# one ncu capture of the default column kernel (16-slice sweep), exported to CSV
SWEEP_SLICES=16 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cols_conv -c 1 -o gpurun_out/k2_cur -f python tools/toeplitz_sweep.py > /dev/null 2>&1
ncu -i gpurun_out/k2_cur.ncu-rep --page raw --csv > gpurun_out/k2_cur.raw.csv 2>/dev/null
ncu -i gpurun_out/k2_cur.ncu-rep --page source --csv --print-source sass > gpurun_out/k2_cur.source.csv 2>/dev/null
gzip -f gpurun_out/k2_cur.source.csv
rm -f gpurun_out/k2_cur.ncu-rep
