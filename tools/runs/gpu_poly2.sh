mkdir -p gpurun_out
for v in "" p3 p4 p5 p6; do
  BFLA_LIB_VARIANT=$v timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/poly_${v:-base}.json 2>&1
done
