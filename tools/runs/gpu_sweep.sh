mkdir -p gpurun_out
timeout 600 python tools/sweep.py --set c2 --out gpurun_out/r1_sweep_c2.md > gpurun_out/sweep_c2.log 2>&1
timeout 1500 python tools/sweep.py --set c5 --out gpurun_out/r1_sweep_c5.md > gpurun_out/sweep_c5.log 2>&1
