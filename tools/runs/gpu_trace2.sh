mkdir -p gpurun_out
timeout 300 python tools/attn_trace.py --out gpurun_out/trace_sparse.json > gpurun_out/trace_sparse.txt 2>&1
cp gpurun_out/attn_trace_cta0.npz gpurun_out/trace_sparse.npz
timeout 300 python tools/attn_trace.py --dense --out gpurun_out/trace_dense.json > gpurun_out/trace_dense.txt 2>&1
cp gpurun_out/attn_trace_cta0.npz gpurun_out/trace_dense.npz
