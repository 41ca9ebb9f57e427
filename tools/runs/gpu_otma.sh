mkdir -p gpurun_out
for rep in 1 2; do for v in 1 0; do
BFLA_OTMA=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/otma_${v}_$rep.json 2>&1
done; done
