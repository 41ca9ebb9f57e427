# session 3 call 10: same-box A/B: base (round-2 head) / product (csz 2) / exp csz 1 / gf (compile-time csz 1)
mkdir -p gpurun_out
for rep in 1 2; do for n in 131072 32768; do
  timeout 300 python tools/s1_timing.py --n $n --variant base >> gpurun_out/r3j_s1.txt 2>&1
  timeout 300 python tools/s1_timing.py --n $n >> gpurun_out/r3j_s1.txt 2>&1
  BFLA_S1_CLUSTER=1 timeout 300 python tools/s1_timing.py --n $n --variant exp >> gpurun_out/r3j_s1.txt 2>&1
  timeout 300 python tools/s1_timing.py --n $n --variant gf >> gpurun_out/r3j_s1.txt 2>&1
done; done
echo done
