mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/band_tests.txt 2>&1; echo "exit $?" >> gpurun_out/band_tests.txt
if grep -q "exit 0" gpurun_out/band_tests.txt; then
timeout 1500 python tools/sweep.py --set c5 --out gpurun_out/r1_sweep_c5b.md > gpurun_out/sweep_c5b.log 2>&1
fi
