mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_attn2 -s 3 -c 1 -o gpurun_out/prof_attn_r1b python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_attn_r1b.log 2>&1
