mkdir -p gpurun_out
timeout 300 python tools/attn_trace.py --out gpurun_out/trace_otma.json > gpurun_out/trace_otma.txt 2>&1
cp gpurun_out/attn_trace_cta0.npz gpurun_out/trace_otma.npz
