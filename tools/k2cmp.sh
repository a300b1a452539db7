for v in nb1 nb1p; do
TF_K2=$v timeout 600 ncu --set full --clock-control none -k regex:k_cols_conv -c 1 -o gpurun_out/k2_$v -f python tools/toeplitz_sweep.py > /dev/null 2>&1
ncu -i gpurun_out/k2_$v.ncu-rep --page raw --csv > gpurun_out/k2_$v.raw.csv 2>/dev/null
rm -f gpurun_out/k2_$v.ncu-rep
done
