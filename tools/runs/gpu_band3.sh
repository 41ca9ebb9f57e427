mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/band_tests.txt 2>&1; echo "exit $?" >> gpurun_out/band_tests.txt
if grep -q "exit 0" gpurun_out/band_tests.txt; then
bash tools/runs/gpu_s1brk.sh
for n in 32768 131072; do timeout 300 python tools/s1_timing.py --n $n >> gpurun_out/s1t.txt 2>&1; done
timeout 300 python tools/s1_timing.py --n 131072 --hq 16 --d 256 >> gpurun_out/s1t.txt 2>&1
fi
