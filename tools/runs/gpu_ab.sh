set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3 > gpurun_out/ab_tests.txt
timeout 300 python tools/attn_trace.py --out gpurun_out/trace_sparse.json > gpurun_out/trace_sparse.txt 2>&1
for mf in 1 0; do
  BFLA_MAXFIRST=$mf timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ab_mf$mf.json 2>&1
  BFLA_MAXFIRST=$mf timeout 600 python bench.py --workload llama8b-128k --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_mf${mf}_128k.json 2>&1
done
