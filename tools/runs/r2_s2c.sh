# session 2 call 3: default bench (varlen_mix point), attention timeline (dense + sparse), cuDNN SDPA launch config
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/s2c_bench.json 2> gpurun_out/s2c_bench.err
timeout 120 python tools/attn_trace.py --dense --out gpurun_out/s2c_trace_dense.json > gpurun_out/s2c_trace_dense.txt 2>&1
cp gpurun_out/attn_trace_cta0.npz gpurun_out/s2c_trace_dense_cta0.npz 2>/dev/null
timeout 120 python tools/attn_trace.py --out gpurun_out/s2c_trace_sparse.json > gpurun_out/s2c_trace_sparse.txt 2>&1
cp gpurun_out/attn_trace_cta0.npz gpurun_out/s2c_trace_sparse_cta0.npz 2>/dev/null
timeout 300 ncu --section LaunchStats --section Occupancy --section SpeedOfLight --section ComputeWorkloadAnalysis --section WarpStateStats --clock-control none -k regex:"fmha|sm100|cudnn|flash" -c 1 python tools/sdpa_probe.py --backend cudnn --reps 2 > gpurun_out/s2c_sdpa_ncu.txt 2>&1
echo done
