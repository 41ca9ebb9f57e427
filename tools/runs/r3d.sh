# session 3 call 4: Gram-free scores with LDS + proxy fence before the stage release
mkdir -p gpurun_out
timeout 600 python tools/norm_check.py > gpurun_out/r3d_norms.txt 2>&1
timeout 600 python tools/norm_check.py >> gpurun_out/r3d_norms.txt 2>&1
for n in 32768 131072 8192 4096; do timeout 300 python tools/s1_timing.py --n $n >> gpurun_out/r3d_s1.txt 2>&1; done
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r3d_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3d_tests.txt
echo done
