mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/s2_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/s2_tests.txt
python tools/stats_cost.py > gpurun_out/s2_cost.txt 2>&1; python tools/stats_cost.py 131072 >> gpurun_out/s2_cost.txt 2>&1
