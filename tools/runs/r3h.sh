# session 3 call 8 (128-row B boxes): score-kernel clusters (B stages multicast over the query heads of a KV group): A/B csz 1/2/4/8
mkdir -p gpurun_out
timeout 600 python tools/norm_check.py > gpurun_out/r3h_norms.txt 2>&1
for n in 32768 131072; do
for env in "BFLA_S1_CLUSTER=1" "BFLA_S1_CLUSTER=2" "BFLA_S1_CLUSTER=4" "BFLA_S1_CLUSTER=8" "BFLA_S1_CLUSTER=1 BFLA_TC_SPLITS=1" "BFLA_S1_CLUSTER=2 BFLA_TC_SPLITS=1" "BFLA_S1_CLUSTER=4 BFLA_TC_SPLITS=1"; do
  env $env timeout 300 python tools/s1_timing.py --n $n --variant exp >> gpurun_out/r3h_s1.txt 2>&1
done; done
timeout 300 python tools/s1_timing.py --n 65536 --hq 64 --hkv 8 >> gpurun_out/r3h_s1.txt 2>&1
BFLA_S1_CLUSTER=8 timeout 300 python tools/s1_timing.py --n 65536 --hq 64 --hkv 8 --variant exp >> gpurun_out/r3h_s1.txt 2>&1
BFLA_S1_CLUSTER=1 timeout 300 python tools/s1_timing.py --n 65536 --hq 64 --hkv 8 --variant exp >> gpurun_out/r3h_s1.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3h_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3h_tests.txt
echo done
