mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1v16_smoke.txt 2>&1
timeout 900 python bench.py --steps 30 --warmup 3 > gpurun_out/r1v16_bench_llama8b-32k.json 2> gpurun_out/r1v16_bench_llama8b-32k.err
for w in llama8b-128k qwen32b-64k-paged gemma-d256-32k; do
  timeout 600 python bench.py --workload $w --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/r1v16_bench_$w.json 2> gpurun_out/r1v16_bench_$w.err
done
bash tools/runs/gpu_launches.sh r1v16_llama32k
