# session 3 call 9: same-box A/B: round-2 head (base) vs Gram-free + cluster (product csz 2, exp csz 1)
mkdir -p gpurun_out
for rep in 1 2; do for n in 32768 131072; do
  timeout 300 python tools/s1_timing.py --n $n --variant base >> gpurun_out/r3i_s1.txt 2>&1
  timeout 300 python tools/s1_timing.py --n $n >> gpurun_out/r3i_s1.txt 2>&1
  BFLA_S1_CLUSTER=1 timeout 300 python tools/s1_timing.py --n $n --variant exp >> gpurun_out/r3i_s1.txt 2>&1
  BFLA_S1_CLUSTER=1 BFLA_TC_SPLITS=1 timeout 300 python tools/s1_timing.py --n $n --variant exp >> gpurun_out/r3i_s1.txt 2>&1
  BFLA_TC_SPLITS=1 timeout 300 python tools/s1_timing.py --n $n --variant exp >> gpurun_out/r3i_s1.txt 2>&1
done; done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_throttle_reasons.active --format=csv >> gpurun_out/r3i_s1.txt
echo done
