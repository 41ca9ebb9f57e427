mkdir -p gpurun_out
for p in 0 3 4 5; do BFLA_POLY=$p timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/poly$p.json 2>&1; done
for p in 0 3 4; do BFLA_POLY=$p timeout 600 python bench.py --workload llama8b-128k --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/poly${p}_128k.json 2>&1; done
