mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/qn_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/qn_tests.txt
( python tools/s1_timing.py
BFLA_QNORM_KERNEL=1 python tools/s1_timing.py
python tools/s1_timing.py --n 131072 --reps 5
BFLA_QNORM_KERNEL=1 python tools/s1_timing.py --n 131072 --reps 5 ) > gpurun_out/qn_s1t.txt 2>&1
bash tools/runs/gpu_launches.sh qn
