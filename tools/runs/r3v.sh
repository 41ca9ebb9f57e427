# session 3 call 22: split-K factor A/B with the current score kernel (cluster pairs, reduce finish)
mkdir -p gpurun_out
for n in 32768 16384 8192; do
  timeout 300 python tools/s1_timing.py --n $n >> gpurun_out/r3v_s1.txt 2>&1
  for s in 1 2 3 4 6 8; do BFLA_TC_SPLITS=$s timeout 300 python tools/s1_timing.py --n $n --variant exp >> gpurun_out/r3v_s1.txt 2>&1; done
  for s in 2 3 4; do BFLA_TC_SPLITS=$s BFLA_S1_FUSED_SPLIT=1 timeout 300 python tools/s1_timing.py --n $n --variant exp >> gpurun_out/r3v_s1.txt 2>&1; done
done
echo done
