# round-1 final measurement pass (current tree)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r1v12_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/r1v12_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1v12_smoke.txt 2>&1
timeout 900 python bench.py --steps 30 --warmup 3 > gpurun_out/r1v12_bench_llama8b-32k.json 2> gpurun_out/r1v12_bench_llama8b-32k.err
for w in llama8b-128k qwen32b-64k-paged gemma-d256-32k; do
  timeout 600 python bench.py --workload $w --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/r1v12_bench_$w.json 2> gpurun_out/r1v12_bench_$w.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r1v12_bench_reference.json 2> gpurun_out/r1v12_bench_reference.err
bash tools/runs/gpu_launches.sh r1v12_llama32k
bash tools/runs/gpu_launches.sh r1v12_llama128k --workload llama8b-128k
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_attn2|k_s1_tc_scores|k_s1_block_norms|k_s1_recompute|k_s1_select|k_s2_expand" -c 7 -o gpurun_out/prof_r1v12 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_r1v12.log 2>&1
timeout 900 python tools/mask_sweep.py --out gpurun_out/tabmask_sweep_v12.md > gpurun_out/tabmask_sweep_v12.log 2>&1
timeout 600 python tools/sweep.py --set c2 --out gpurun_out/r1v12_sweep_c2.md > gpurun_out/r1v12_sweep_c2.log 2>&1
timeout 1500 python tools/sweep.py --set c5 --out gpurun_out/r1v12_sweep_c5.md > gpurun_out/r1v12_sweep_c5.log 2>&1
