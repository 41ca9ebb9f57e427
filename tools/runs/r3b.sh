# session 3 call 2: Stage-1 scores without the Gram MMA (norms from the A stages) + in-kernel split-K fixup
mkdir -p gpurun_out
for n in 32768 131072; do timeout 300 python tools/s1_timing.py --n $n >> gpurun_out/r3b_s1.txt 2>&1; done
timeout 300 python tools/s1_timing.py --n 8192 >> gpurun_out/r3b_s1.txt 2>&1
timeout 300 python tools/s1_timing.py --n 4096 >> gpurun_out/r3b_s1.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3b_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3b_tests.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(s1|s2|attn|paged)" -c 200 --csv --log-file gpurun_out/r3b_launches_32k.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/r3b_ncu32.log 2>&1
echo done
