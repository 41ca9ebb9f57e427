# session 2 call 22: ncu --set full of every hot kernel of the current code (32K default line), launch list
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(s1_tc_scores|s1_select|s1_block_norms|s1_recompute|s1_tc_reduce|s2_expand|attn2)" -c 9 -o gpurun_out/s2y_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/s2y_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(s1|s2|attn|paged)" -c 200 --csv --log-file gpurun_out/s2y_launches_32k.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/s2y_ncu32.log 2>&1
echo done
