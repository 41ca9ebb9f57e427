# session 3 call 11: same-box A/B: base / Gram+cluster2+fused split (product) / its knobs / norm-warps variant
mkdir -p gpurun_out
timeout 600 python tools/norm_check.py > gpurun_out/r3k_norms.txt 2>&1
for rep in 1 2; do for n in 32768 131072; do
  timeout 300 python tools/s1_timing.py --n $n --variant base >> gpurun_out/r3k_s1.txt 2>&1
  timeout 300 python tools/s1_timing.py --n $n >> gpurun_out/r3k_s1.txt 2>&1
  BFLA_S1_CLUSTER=1 timeout 300 python tools/s1_timing.py --n $n --variant exp >> gpurun_out/r3k_s1.txt 2>&1
  BFLA_TC_SPLITS=1 timeout 300 python tools/s1_timing.py --n $n --variant exp >> gpurun_out/r3k_s1.txt 2>&1
  BFLA_S1_CLUSTER=4 timeout 300 python tools/s1_timing.py --n $n --variant exp >> gpurun_out/r3k_s1.txt 2>&1
  timeout 300 python tools/s1_timing.py --n $n --variant nw >> gpurun_out/r3k_s1.txt 2>&1
done; done
for n in 4096 8192 16384; do
  timeout 300 python tools/s1_timing.py --n $n --variant base >> gpurun_out/r3k_s1.txt 2>&1
  timeout 300 python tools/s1_timing.py --n $n >> gpurun_out/r3k_s1.txt 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3k_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3k_tests.txt
echo done
