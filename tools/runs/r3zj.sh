# session 3 call 36: pair-kernel stage count A/B (5 / 6 / 7) + ncu --set full of the pair kernel (32K, 128K)
mkdir -p gpurun_out
for rep in 1 2; do for n in 32768 131072; do
  timeout 120 python tools/s1_timing.py --n $n >> gpurun_out/r3zj_s1.txt 2>&1
  timeout 120 python tools/s1_timing.py --n $n --variant pst7 >> gpurun_out/r3zj_s1.txt 2>&1
  timeout 120 python tools/s1_timing.py --n $n --variant pst5 >> gpurun_out/r3zj_s1.txt 2>&1
done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_s1_tc_scores" -c 1 -o gpurun_out/r3zj_pair32 python tools/s1_timing.py --n 32768 --reps 1 > gpurun_out/r3zj.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_s1_tc_scores" -c 1 -o gpurun_out/r3zj_pair128 python tools/s1_timing.py --n 131072 --reps 1 >> gpurun_out/r3zj.log 2>&1
echo done
