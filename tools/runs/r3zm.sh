# session 3 call 40: reduce kernel with all columns' loads in flight and a max pyramid: A/B + GPU suite
mkdir -p gpurun_out
for rep in 1 2; do for n in 32768 16384; do
  timeout 120 python tools/s1_timing.py --n $n --variant prev >> gpurun_out/r3zm_s1.txt 2>&1
  timeout 120 python tools/s1_timing.py --n $n >> gpurun_out/r3zm_s1.txt 2>&1
done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_s1_tc_reduce" -c 6 --csv --log-file gpurun_out/r3zm_red.csv python tools/s1_timing.py --n 32768 --reps 2 > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3zm_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3zm_tests.txt
echo done
