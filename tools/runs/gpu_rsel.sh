mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/rsel_tests.txt 2>&1; echo "exit $?" >> gpurun_out/rsel_tests.txt
if grep -q "exit 0" gpurun_out/rsel_tests.txt; then
bash tools/runs/gpu_s1brk.sh
for r in 0.05 0.1 0.4; do timeout 300 python tools/s1_timing.py --n 131072 --ratio $r >> gpurun_out/rsel.txt 2>&1; done
timeout 300 python tools/s1_timing.py --n 32768 >> gpurun_out/rsel.txt 2>&1
fi
