# round 2 baseline: bench on this pool's box + cuDNN SDPA kernel structure (ncu) for comparison
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b_build.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
timeout 120 python tools/sdpa_probe.py --backend cudnn > gpurun_out/r2b_sdpa.txt 2>&1
timeout 120 python tools/sdpa_probe.py --backend flash >> gpurun_out/r2b_sdpa.txt 2>&1
timeout 400 ncu --set full --clock-control none -k regex:"cudnn|sm100|fmha|flash" -c 1 -o gpurun_out/r2b_sdpa_prof python tools/sdpa_probe.py --backend cudnn --reps 1 > gpurun_out/r2b_sdpa_ncu.txt 2>&1
echo done
