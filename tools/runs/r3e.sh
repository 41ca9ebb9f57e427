# session 3 call 5: Stage-1 A/B at 32K/128K: q norms in the score kernel vs the HBM kernel, split-K factor
mkdir -p gpurun_out
for n in 32768 131072; do
for env in "" "BFLA_QNORM_KERNEL=1" "BFLA_TC_SPLITS=1" "BFLA_TC_SPLITS=1 BFLA_QNORM_KERNEL=1" "BFLA_TC_SPLITS=3" "BFLA_TC_SPLITS=4"; do
  env $env timeout 300 python tools/s1_timing.py --n $n --variant exp >> gpurun_out/r3e_s1.txt 2>&1
done; done
echo done
