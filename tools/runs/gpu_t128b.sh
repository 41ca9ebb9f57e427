mkdir -p gpurun_out
for w in llama8b-32k llama8b-128k gemma-d256-32k; do
  timeout 600 python bench.py --workload $w --tile 128 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/t128_bench_$w.json 2> gpurun_out/t128_bench_$w.err
done
