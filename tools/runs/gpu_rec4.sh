mkdir -p gpurun_out
bash tools/runs/gpu_launches.sh rec4
BFLA_RECOMPUTE_GLOBAL=1 bash tools/runs/gpu_launches.sh rec4g
