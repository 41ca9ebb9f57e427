mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/otma_tests.txt 2>&1
for o in 1 0; do BFLA_OTMA=$o timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/otma$o.json 2>&1; done
for o in 1 0; do BFLA_OTMA=$o timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/otma${o}b.json 2>&1; done
BFLA_OTMA=1 timeout 600 python bench.py --workload llama8b-128k --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/otma1_128k.json 2>&1
BFLA_OTMA=1 timeout 600 python bench.py --workload qwen32b-64k-paged --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/otma1_qwen.json 2>&1
timeout 300 python tools/attn_trace.py --out gpurun_out/trace_otma.json > gpurun_out/trace_otma.txt 2>&1
cp gpurun_out/attn_trace_cta0.npz gpurun_out/trace_otma.npz
