mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "certification_norms or fast_scores or shapes or tiny or head_dim or paged" > gpurun_out/rec3_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/rec3_tests.txt
python tools/s1_timing.py > gpurun_out/rec3_s1t.txt 2>&1
BFLA_RECOMPUTE_GLOBAL=1 python tools/s1_timing.py >> gpurun_out/rec3_s1t.txt 2>&1
BFLA_TAU_SCALE=1e-6 python tools/s1_timing.py >> gpurun_out/rec3_s1t.txt 2>&1
BFLA_TAU_SCALE=4 python tools/s1_timing.py >> gpurun_out/rec3_s1t.txt 2>&1
python tools/s1_timing.py --n 131072 --reps 5 >> gpurun_out/rec3_s1t.txt 2>&1
