# session 3 call 23: split-K factor from the live tile count — Stage-1 sizes, full GPU suite
mkdir -p gpurun_out
for n in 4096 8192 16384 32768 65536 131072; do timeout 300 python tools/s1_timing.py --n $n >> gpurun_out/r3w_s1.txt 2>&1; done
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r3w_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3w_tests.txt
echo done
