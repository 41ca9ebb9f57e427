# session 3 call 19: split-K reduce kernel granularity A/B (64 / 32 / 16 key-group columns per CTA)
mkdir -p gpurun_out
for rep in 1 2; do for n in 32768 16384; do
  timeout 300 python tools/s1_timing.py --n $n >> gpurun_out/r3s_s1.txt 2>&1
  timeout 300 python tools/s1_timing.py --n $n --variant rc32 >> gpurun_out/r3s_s1.txt 2>&1
  timeout 300 python tools/s1_timing.py --n $n --variant rc16 >> gpurun_out/r3s_s1.txt 2>&1
done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_s1" -c 40 --csv --log-file gpurun_out/r3s_l64.csv python tools/s1_timing.py --n 32768 --reps 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_s1" -c 40 --csv --log-file gpurun_out/r3s_l16.csv python tools/s1_timing.py --n 32768 --reps 3 --variant rc16 > /dev/null 2>&1
echo done
