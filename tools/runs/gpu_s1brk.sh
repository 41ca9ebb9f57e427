mkdir -p gpurun_out
ncu --kernel-name regex:k_ --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s1brk_r01.csv timeout 900 python tools/s1_timing.py --n 131072 --hq 16 --hkv 8 --d 256 --ratio 0.1 --reps 2 > gpurun_out/s1brk.txt 2>&1
ncu --kernel-name regex:k_ --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s1brk_r01_d128.csv timeout 900 python tools/s1_timing.py --n 131072 --hq 32 --hkv 8 --d 128 --ratio 0.1 --reps 2 >> gpurun_out/s1brk.txt 2>&1
python tools/launch_summary.py gpurun_out/s1brk_r01.csv > gpurun_out/s1brk_sum.txt 2>&1
python tools/launch_summary.py gpurun_out/s1brk_r01_d128.csv >> gpurun_out/s1brk_sum.txt 2>&1
