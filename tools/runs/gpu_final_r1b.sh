# round-1 measurement pass (current tree): bench lines for every workload, launch lists, ncu --set full of the hot kernels
mkdir -p gpurun_out
timeout 900 python bench.py --steps 30 --warmup 3 > gpurun_out/r1v10_bench_llama8b-32k.json 2> gpurun_out/r1v10_bench_llama8b-32k.err
for w in llama8b-128k qwen32b-64k-paged gemma-d256-32k; do
  timeout 600 python bench.py --workload $w --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/r1v10_bench_$w.json 2> gpurun_out/r1v10_bench_$w.err
done
bash tools/runs/gpu_launches.sh r1v10_llama32k
bash tools/runs/gpu_launches.sh r1v10_llama128k --workload llama8b-128k
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_attn2|k_s1_tc_scores|k_s1_block_norms|k_s1_recompute|k_s1_select|k_s2_expand" -c 7 -o gpurun_out/prof_r1v10 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_r1v10.log 2>&1
