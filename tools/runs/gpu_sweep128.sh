mkdir -p gpurun_out
timeout 1500 python tools/sweep.py --set c5 --tile 128 --out gpurun_out/r1v12_sweep_c5_t128.md > gpurun_out/r1v12_sweep_c5_t128.log 2>&1
