mkdir -p gpurun_out
for rep in 1 2; do for v in "" pf0 pf2 pf5; do
BFLA_LIB_VARIANT=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/pf_${v:-base}_$rep.json 2>&1
done; done
