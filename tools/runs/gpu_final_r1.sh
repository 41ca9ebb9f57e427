# round-1 measurement pass: bench lines for every workload, launch lists, ncu --set full of the hot kernels
mkdir -p gpurun_out
for w in llama8b-128k qwen32b-64k-paged gemma-d256-32k; do
  timeout 600 python bench.py --workload $w --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/r1v9_bench_$w.json 2> gpurun_out/r1v9_bench_$w.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r1v9_bench_reference.json 2> gpurun_out/r1v9_bench_reference.err
bash tools/runs/gpu_launches.sh r1v9_llama32k
bash tools/runs/gpu_launches.sh r1v9_llama128k --workload llama8b-128k
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_attn2|k_s1_tc_scores|k_s1_block_norms|k_s1_recompute|k_s1_select|k_s2_expand" -c 7 -o gpurun_out/prof_r1v9 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_r1v9.log 2>&1
