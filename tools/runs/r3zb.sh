# session 3 call 28: K-norm kernel as a one-CTA-per-SM grid-stride kernel beside the score kernel: bench + s1 timing + tests
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r3zb_bench.json 2> gpurun_out/r3zb_bench.err
for n in 32768 131072 8192; do timeout 300 python tools/s1_timing.py --n $n >> gpurun_out/r3zb_s1.txt 2>&1; done
timeout 1500 python -m pytest tests -m gpu -q -x -k "norm or cert or fullsize or shapes or varlen" > gpurun_out/r3zb_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3zb_tests.txt
echo done
