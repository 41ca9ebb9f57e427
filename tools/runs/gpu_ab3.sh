mkdir -p gpurun_out
for rep in 1 2; do for v in "" r88 noqr; do
  BFLA_LIB_VARIANT=$v timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ab3_${v:-base}_$rep.json 2>&1
done; done
for v in "" r88 noqr; do
  BFLA_LIB_VARIANT=$v timeout 600 python bench.py --workload llama8b-128k --steps 6 --warmup 2 --no-cpu-baseline > gpurun_out/ab3_${v:-base}_128k.json 2>&1
done
