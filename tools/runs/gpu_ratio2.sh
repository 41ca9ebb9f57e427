mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k "ratio or mean_pool or fast_scores or tiny" > gpurun_out/ratio2_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/ratio2_tests.txt
( for r in 0.02 0.1 0.4; do python tools/s1_timing.py --ratio $r --reps 5; done ) > gpurun_out/ratio2_s1t.txt 2>&1
