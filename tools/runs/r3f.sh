# session 3 call 6: ncu --set full of the Gram-free score kernel at 32K (split 1 and 2) and 128K
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_s1_tc_scores" -c 1 -o gpurun_out/r3f_s1_32k python tools/s1_timing.py --n 32768 --reps 1 > gpurun_out/r3f_ncu.log 2>&1
BFLA_TC_SPLITS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_s1_tc_scores" -c 1 -o gpurun_out/r3f_s1_32k_split1 python tools/s1_timing.py --n 32768 --reps 1 --variant exp >> gpurun_out/r3f_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_s1_tc_scores" -c 1 -o gpurun_out/r3f_s1_128k python tools/s1_timing.py --n 131072 --reps 1 >> gpurun_out/r3f_ncu.log 2>&1
echo done
