# session 3 call 13: defaults = norm warps + cluster 2 + split finish by grid size; norms, GPU suite, timings
mkdir -p gpurun_out
timeout 600 python tools/norm_check.py > gpurun_out/r3m_norms.txt 2>&1
for n in 4096 8192 16384 32768 65536 131072; do timeout 300 python tools/s1_timing.py --n $n >> gpurun_out/r3m_s1.txt 2>&1; timeout 300 python tools/s1_timing.py --n $n --variant base >> gpurun_out/r3m_s1.txt 2>&1; done
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r3m_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3m_tests.txt
echo done
