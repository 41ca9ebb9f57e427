mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/band_tests.txt 2>&1; echo "exit $?" >> gpurun_out/band_tests.txt
if grep -q "exit 0" gpurun_out/band_tests.txt; then
bash tools/runs/gpu_s1brk.sh
fi
