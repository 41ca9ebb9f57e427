# round-1 final measurement pass (r1_v14)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r1v14_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r1v14_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1v14_smoke.txt 2>&1
timeout 900 python bench.py --steps 30 --warmup 3 > gpurun_out/r1v14_bench_llama8b-32k.json 2> gpurun_out/r1v14_bench_llama8b-32k.err
for w in llama8b-128k qwen32b-64k-paged gemma-d256-32k; do
  timeout 600 python bench.py --workload $w --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/r1v14_bench_$w.json 2> gpurun_out/r1v14_bench_$w.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r1v14_bench_reference.json 2> gpurun_out/r1v14_bench_reference.err
bash tools/runs/gpu_launches.sh r1v14_llama32k
bash tools/runs/gpu_launches.sh r1v14_llama128k --workload llama8b-128k
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_attn2|k_s1_tc_scores|k_s1_tc_reduce|k_s1_block_norms|k_s1_recompute|k_s1_select|k_s2_expand" -c 8 -o gpurun_out/prof_r1v14 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_r1v14.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize_cases.py > gpurun_out/r1_sanitizer4_$tool.log 2>&1
  echo "exit=$?" >> gpurun_out/r1_sanitizer4_$tool.log
done
timeout 600 python tools/sweep.py --set c2 --out gpurun_out/r1v14_sweep_c2.md > gpurun_out/r1v14_sweep_c2.log 2>&1
timeout 1500 python tools/sweep.py --set c5 --out gpurun_out/r1v14_sweep_c5.md > gpurun_out/r1v14_sweep_c5.log 2>&1
