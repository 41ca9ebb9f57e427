# session 3 call 37: pair kernel — the peer's A counts at the leader outside the query-norm tiles (no forward): A/B + tests
mkdir -p gpurun_out
for rep in 1 2; do for n in 32768 131072 65536; do
  timeout 120 python tools/s1_timing.py --n $n --variant prev >> gpurun_out/r3zk_s1.txt 2>&1
  timeout 120 python tools/s1_timing.py --n $n >> gpurun_out/r3zk_s1.txt 2>&1
done; done
timeout 300 python tools/norm_check.py > gpurun_out/r3zk_norms.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3zk_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3zk_tests.txt
echo done
