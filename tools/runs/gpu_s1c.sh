mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "certification_norms or fast_scores or shapes or tiny_structured" > gpurun_out/s1c_tests.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/s1c_bench.json 2>&1
bash tools/runs/gpu_launches.sh s1c
