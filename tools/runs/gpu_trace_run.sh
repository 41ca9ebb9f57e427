mkdir -p gpurun_out
timeout 300 python tools/attn_trace.py --out gpurun_out/trace_sparse.json > gpurun_out/trace_sparse.txt 2>&1
cp gpurun_out/attn_trace_cta0.npz gpurun_out/trace_opt0.npz
BFLA_ATTN_OPTS=1 timeout 300 python tools/attn_trace.py --out gpurun_out/trace_sparse1.json > gpurun_out/trace_sparse1.txt 2>&1
cp gpurun_out/attn_trace_cta0.npz gpurun_out/trace_opt1.npz
for o in 0 1; do BFLA_ATTN_OPTS=$o timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ab_opt$o.json 2>&1; done
