mkdir -p gpurun_out
for rep in 1 2; do
for sp in 1 2 3 4; do
  echo "splits=$sp" >> gpurun_out/splits_ab.txt
  BFLA_TC_SPLITS=$sp timeout 300 python tools/s1_timing.py --n 32768 >> gpurun_out/splits_ab.txt 2>&1
  BFLA_TC_SPLITS=$sp timeout 300 python tools/s1_timing.py --n 65536 --hq 64 >> gpurun_out/splits_ab.txt 2>&1
done
done
