# session 3 call 15: bench line on the new Stage 1, launch list 32K, ncu --set full of the score kernel (32K, 128K)
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r3o_bench.json 2> gpurun_out/r3o_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(s1|s2|attn|paged)" -c 200 --csv --log-file gpurun_out/r3o_launches_32k.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/r3o_ncu32.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_s1_tc_scores" -c 1 -o gpurun_out/r3o_s1_32k python tools/s1_timing.py --n 32768 --reps 1 > gpurun_out/r3o_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_s1_tc_scores" -c 1 -o gpurun_out/r3o_s1_128k python tools/s1_timing.py --n 131072 --reps 1 >> gpurun_out/r3o_ncu.log 2>&1
echo done
