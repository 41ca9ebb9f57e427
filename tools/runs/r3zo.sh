# session 3 call 43: after removing the Gram / no-cluster A/B code paths: GPU suite, norm check, timing
mkdir -p gpurun_out
timeout 300 python tools/norm_check.py > gpurun_out/r3zo_norms.txt 2>&1
for n in 8192 32768 131072; do timeout 120 python tools/s1_timing.py --n $n >> gpurun_out/r3zo_s1.txt 2>&1; done
BFLA_S1_PAIR=0 timeout 120 python tools/s1_timing.py --n 32768 --variant exp >> gpurun_out/r3zo_s1.txt 2>&1
BFLA_S1_CLUSTER=1 timeout 120 python tools/s1_timing.py --n 32768 --variant exp >> gpurun_out/r3zo_s1.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r3zo_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3zo_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3zo_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r3zo_smoke.txt
echo done
