# session 3 call 24: canonical Z sum with 16-byte loads in k_s1_select (A/B vs the previous build) + GPU suite
mkdir -p gpurun_out
for rep in 1 2; do for n in 131072 32768; do
  timeout 300 python tools/s1_timing.py --n $n --variant prev >> gpurun_out/r3x_s1.txt 2>&1
  timeout 300 python tools/s1_timing.py --n $n >> gpurun_out/r3x_s1.txt 2>&1
done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_s1" -c 12 --csv --log-file gpurun_out/r3x_l128.csv python tools/s1_timing.py --n 131072 --reps 1 > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3x_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3x_tests.txt
echo done
