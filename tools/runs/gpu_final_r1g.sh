mkdir -p gpurun_out
bash tools/runs/gpu_sanitize.sh
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r1v15_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r1v15_tests.txt
timeout 900 python bench.py --steps 30 --warmup 3 > gpurun_out/r1v15_bench_llama8b-32k.json 2> gpurun_out/r1v15_bench_llama8b-32k.err
timeout 600 python bench.py --workload gemma-d256-32k --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/r1v15_bench_gemma-d256-32k.json 2> gpurun_out/r1v15_bench_gemma-d256-32k.err
