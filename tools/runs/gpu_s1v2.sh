mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_norms or fast_scores or shapes or tiny_structured" > gpurun_out/s1v2_tests.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/s1v2_bench.json 2>&1
BFLA_S1_V1=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/s1v1_bench.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/s1v2_launches.csv 2>&1
