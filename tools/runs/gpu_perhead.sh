mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/perhead_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/perhead_tests.txt
timeout 900 python tools/mask_sweep.py --out gpurun_out/tabmask_sweep.md > gpurun_out/tabmask_sweep.log 2>&1
