# session 3 call 12: same-box A/B: split finish (fused/reduce) x cluster x query-norm source
mkdir -p gpurun_out
for rep in 1 2; do for n in 32768 131072 8192; do
  timeout 300 python tools/s1_timing.py --n $n --variant base >> gpurun_out/r3l_s1.txt 2>&1
  timeout 300 python tools/s1_timing.py --n $n >> gpurun_out/r3l_s1.txt 2>&1
  for v in exp nw; do for env in "BFLA_S1_CLUSTER=1 BFLA_S1_FUSED_SPLIT=0" "BFLA_S1_CLUSTER=2 BFLA_S1_FUSED_SPLIT=0" "BFLA_S1_CLUSTER=1 BFLA_S1_FUSED_SPLIT=1" "BFLA_S1_CLUSTER=2 BFLA_S1_FUSED_SPLIT=1"; do
    env $env timeout 300 python tools/s1_timing.py --n $n --variant $v >> gpurun_out/r3l_s1.txt 2>&1
  done; done
done; done
echo done
