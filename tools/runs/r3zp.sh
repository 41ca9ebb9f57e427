# session 3 call 44: selection kernel with redux.sync 64-bit warp max: A/B (block_mask + bench) + GPU suite
mkdir -p gpurun_out
for rep in 1 2; do for n in 32768 131072; do
  timeout 120 python tools/s1_timing.py --n $n --variant prev >> gpurun_out/r3zp_s1.txt 2>&1
  timeout 120 python tools/s1_timing.py --n $n >> gpurun_out/r3zp_s1.txt 2>&1
  timeout 120 python tools/s1_timing.py --n $n --ratio 0.1 --variant prev >> gpurun_out/r3zp_s1.txt 2>&1
  timeout 120 python tools/s1_timing.py --n $n --ratio 0.1 >> gpurun_out/r3zp_s1.txt 2>&1
done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_s1_select" -c 8 --csv --log-file gpurun_out/r3zp_sel.csv python tools/s1_timing.py --n 32768 --reps 2 > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r3zp_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3zp_tests.txt
echo done
