# session 3 call 25: graph-captured bench, reference arm, varlen/chunked workloads on the session-3 Stage 1
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 --graph 1 --no-cpu-baseline --extra-128k 0 > gpurun_out/r3y_bench_graph.json 2> gpurun_out/r3y_bench_graph.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r3y_ref.json 2> gpurun_out/r3y_ref.err
for wl in qwen32b-64k-paged gemma-d256-32k; do timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/r3y_bench_$wl.json 2> gpurun_out/r3y_bench_$wl.err; done
echo done
