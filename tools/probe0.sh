set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/p0_nvsmi.txt 2>&1
free -g > gpurun_out/p0_free.txt; nproc >> gpurun_out/p0_free.txt; lscpu | head -20 >> gpurun_out/p0_free.txt
python -c "import torch; p=torch.cuda.get_device_properties(0); print(p.total_memory, torch.cuda.mem_get_info())" > gpurun_out/p0_mem.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/p0_bench.json 2> gpurun_out/p0_bench.err
