mkdir -p gpurun_out
BFLA_SMX=2 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/split_tests.txt 2>&1
for v in 1 2; do BFLA_SMX=$v timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/smx$v.json 2>&1; done
for v in 1 2; do BFLA_SMX=$v timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/smx${v}b.json 2>&1; done
for v in 1 2; do BFLA_SMX=$v timeout 600 python bench.py --workload llama8b-128k --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/smx${v}_128k.json 2>&1; done
