# session 3 call 39: split-K factor A/B with the CTA-pair score kernel
mkdir -p gpurun_out
for n in 32768 16384 8192 65536; do
  timeout 120 python tools/s1_timing.py --n $n >> gpurun_out/r3zl_s1.txt 2>&1
  for s in 1 2 3 4; do BFLA_TC_SPLITS=$s timeout 120 python tools/s1_timing.py --n $n --variant exp >> gpurun_out/r3zl_s1.txt 2>&1; done
  BFLA_TC_SPLITS=2 BFLA_S1_FUSED_SPLIT=1 timeout 120 python tools/s1_timing.py --n $n --variant exp >> gpurun_out/r3zl_s1.txt 2>&1
done
echo done
