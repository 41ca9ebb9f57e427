mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/rec2_tests.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/rec2_bench.json 2>&1
bash tools/runs/gpu_launches.sh rec2
python tools/s1_timing.py > gpurun_out/rec2_s1t.txt 2>&1
BFLA_TAU_SCALE=4 python tools/s1_timing.py >> gpurun_out/rec2_s1t.txt 2>&1
