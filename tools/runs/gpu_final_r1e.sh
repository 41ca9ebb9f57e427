mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r1v13_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r1v13_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1v13_smoke.txt 2>&1
timeout 900 python bench.py --steps 30 --warmup 3 > gpurun_out/r1v13_bench_llama8b-32k.json 2> gpurun_out/r1v13_bench_llama8b-32k.err
for w in llama8b-128k qwen32b-64k-paged gemma-d256-32k; do
  timeout 600 python bench.py --workload $w --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/r1v13_bench_$w.json 2> gpurun_out/r1v13_bench_$w.err
done
timeout 600 python tools/sweep.py --set c2 --out gpurun_out/r1v13_sweep_c2.md > gpurun_out/r1v13_sweep_c2.log 2>&1
timeout 1500 python tools/sweep.py --set c5 --out gpurun_out/r1v13_sweep_c5.md > gpurun_out/r1v13_sweep_c5.log 2>&1
timeout 1500 python tools/sweep.py --set c5 --tile 128 --out gpurun_out/r1v13_sweep_c5_t128.md > gpurun_out/r1v13_sweep_c5_t128.log 2>&1
