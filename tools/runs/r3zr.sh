# session 3 call 46: pair-kernel grid order with M tiles outermost, bottom rows first (A/B) + parity subset
mkdir -p gpurun_out
for rep in 1 2; do for n in 32768 65536 131072 16384; do
  timeout 120 python tools/s1_timing.py --n $n >> gpurun_out/r3zr_s1.txt 2>&1
  timeout 120 python tools/s1_timing.py --n $n --variant rowdesc >> gpurun_out/r3zr_s1.txt 2>&1
done; done
echo done
