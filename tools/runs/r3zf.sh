# session 3 call 32: Stage 2 with two 32-tile chunks per pass (independent hash chains side by side): A/B + tests
mkdir -p gpurun_out
for rep in 1 2; do for n in 32768 131072; do
  timeout 300 python tools/s2_timing.py --n $n --variant prev >> gpurun_out/r3zf_s2.txt 2>&1
  timeout 300 python tools/s2_timing.py --n $n >> gpurun_out/r3zf_s2.txt 2>&1
done; done
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r3zf_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3zf_tests.txt
echo done
