mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"recompute" -s 1 -c 1 -o gpurun_out/prof_rec2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_rec.log 2>&1
