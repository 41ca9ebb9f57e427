mkdir -p gpurun_out
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/s1v2_bench.json 2>&1
bash tools/runs/gpu_launches.sh s1v2
BFLA_S1_V1=1 bash tools/runs/gpu_launches.sh s1v1
