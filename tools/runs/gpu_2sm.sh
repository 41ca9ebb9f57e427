mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_parity.py -x -q -k "fast_scores" > gpurun_out/2sm_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/2sm_tests.txt
if grep -q "rc=0" gpurun_out/2sm_tests.txt; then
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -k "certification_norms or shapes or tiny or head_dim or paged" >> gpurun_out/2sm_tests.txt 2>&1
echo "rc2=$?" >> gpurun_out/2sm_tests.txt
( python tools/s1_timing.py
BFLA_S1_2SM=0 python tools/s1_timing.py
python tools/s1_timing.py --n 131072 --reps 5
BFLA_S1_2SM=0 python tools/s1_timing.py --n 131072 --reps 5 ) > gpurun_out/2sm_s1t.txt 2>&1
bash tools/runs/gpu_launches.sh 2sm
fi
