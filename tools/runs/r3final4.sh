# session 3 final call 4 (HEAD): full GPU suite, smoke, bench line, launch lists (32K, 128K), ncu --set full of the hot kernels
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r3i_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3i_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3i_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r3i_smoke.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r3i_bench.json 2> gpurun_out/r3i_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(s1|s2|attn|paged)" -c 200 --csv --log-file gpurun_out/r3i_launches_32k.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/r3i_ncu32.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(s1_tc_scores_pair|s1_tc_reduce|s1_select|s1_block_norms|s1_recompute|s2_expand|attn2)" -c 9 -o gpurun_out/r3i_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/r3i_ncufull.log 2>&1
echo done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(s1|s2|attn|paged)" -c 60 --csv --log-file gpurun_out/r3i_launches_128k.csv python bench.py --workload llama8b-128k --steps 2 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/r3i_l.log 2>&1
