# session 3 call 35: CTA-pair score kernel with a relaxed forward arrive: A/B + tests
mkdir -p gpurun_out
for rep in 1 2; do for n in 32768 131072 8192; do
  BFLA_S1_PAIR=0 timeout 120 python tools/s1_timing.py --n $n --variant exp >> gpurun_out/r3zi_s1.txt 2>&1
  timeout 120 python tools/s1_timing.py --n $n >> gpurun_out/r3zi_s1.txt 2>&1
done; done
timeout 300 python tools/norm_check.py > gpurun_out/r3zi_norms.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3zi_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3zi_tests.txt
echo done
