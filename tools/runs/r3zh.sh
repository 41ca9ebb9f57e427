# session 3 call 34: ncu --set full of the CTA-pair score kernel at 32K
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_s1_tc_scores" -c 1 -o gpurun_out/r3zh_pair python tools/s1_timing.py --n 32768 --reps 1 > gpurun_out/r3zh.log 2>&1
echo done
