mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fast_scores or certification_norms or keep_ratio_fast or per_query or tiny or shapes" > gpurun_out/diag_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/diag_tests.txt
( python tools/s1_timing.py; python tools/s1_timing.py --n 131072 --reps 5 ) > gpurun_out/diag_s1t.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/diag_bench.json 2>&1
bash tools/runs/gpu_launches.sh diag
