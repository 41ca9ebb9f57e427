mkdir -p gpurun_out
( python tools/s1_timing.py
BFLA_TAU_SCALE=1e-6 python tools/s1_timing.py
BFLA_TAU_SCALE=4 python tools/s1_timing.py
python tools/s1_timing.py --n 131072 --reps 5
BFLA_TAU_SCALE=1e-6 python tools/s1_timing.py --n 131072 --reps 5 ) > gpurun_out/s1t.txt 2>&1
