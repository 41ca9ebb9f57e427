# session 3 call 26: K-norm kernel launched after the score kernel (A/B vs prev) + launch timeline via nsys-less ncu
mkdir -p gpurun_out
for rep in 1 2; do for n in 32768 131072 65536 8192; do
  timeout 300 python tools/s1_timing.py --n $n --variant prev >> gpurun_out/r3z_s1.txt 2>&1
  timeout 300 python tools/s1_timing.py --n $n >> gpurun_out/r3z_s1.txt 2>&1
done; done
echo done
