# session 3 call 30: launch lists of the Qwen-64K paged and 128K layers (where Stage 1 time goes)
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(s1|s2|attn|paged)" -c 60 --csv --log-file gpurun_out/r3zd_qwen.csv python bench.py --workload qwen32b-64k-paged --steps 2 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/r3zd_q.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(s1|s2|attn|paged)" -c 60 --csv --log-file gpurun_out/r3zd_128k.csv python bench.py --workload llama8b-128k --steps 2 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/r3zd_l.log 2>&1
echo done
