mkdir -p gpurun_out
for rep in 1 2 3; do for v in "" qr1; do
BFLA_LIB_VARIANT=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/qr2_${v:-base}_$rep.json 2>&1
done; done
