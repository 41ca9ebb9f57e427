mkdir -p gpurun_out
( for r in 0.02 0.1 0.4; do python tools/s1_timing.py --ratio $r --reps 5; done
BFLA_SCORES=1 python tools/s1_timing.py --ratio 0.1 --reps 5 ) > gpurun_out/ratio_s1t.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_s1|k_s2" -c 20 --csv python tools/s1_timing.py --ratio 0.1 --reps 1 > gpurun_out/launches_ratio.csv 2>&1
