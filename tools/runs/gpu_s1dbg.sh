mkdir -p gpurun_out
for d in 0 1 2 3; do BFLA_S1_DBG=$d bash tools/runs/gpu_launches.sh dbg$d; done
