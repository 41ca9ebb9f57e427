mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "certification_norms or fast_scores or shapes or tiny or head_dim or paged" > gpurun_out/rec5_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/rec5_tests.txt
( for m in 0 1 2; do BFLA_RECOMPUTE=$m python tools/s1_timing.py; done
BFLA_TAU_SCALE=1e-6 python tools/s1_timing.py
BFLA_TAU_SCALE=4 python tools/s1_timing.py
BFLA_TAU_SCALE=4 BFLA_RECOMPUTE=1 python tools/s1_timing.py
python tools/s1_timing.py --n 131072 --reps 5
BFLA_RECOMPUTE=1 python tools/s1_timing.py --n 131072 --reps 5 ) > gpurun_out/rec5_s1t.txt 2>&1
bash tools/runs/gpu_launches.sh rec5
