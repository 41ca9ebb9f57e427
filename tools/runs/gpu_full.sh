mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1
timeout 600 python bench.py --steps 30 --warmup 3 > gpurun_out/bench_main.json 2>gpurun_out/bench_main.err
