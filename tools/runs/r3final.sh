# session 3 final call: full GPU suite, smoke, bench line, launch lists (32K, 128K), ncu --set full of the hot kernels
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r3f_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3f_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3f_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r3f_smoke.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r3f_bench.json 2> gpurun_out/r3f_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(s1|s2|attn|paged)" -c 200 --csv --log-file gpurun_out/r3f_launches_32k.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/r3f_ncu32.log 2>&1
cp gpurun_out/r3zd_128k.csv gpurun_out/r3f_launches_128k.csv 2>/dev/null || true
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(s1_tc_scores|s1_tc_reduce|s1_select|s1_block_norms|s1_recompute|s2_expand|attn2)" -c 9 -o gpurun_out/r3f_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/r3f_ncufull.log 2>&1
echo done
