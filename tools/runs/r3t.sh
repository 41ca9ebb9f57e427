# session 3 call 20: full GPU suite, smoke, bench line, 32K/128K launch lists on the session-3 code
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r3t_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3t_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3t_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r3t_smoke.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r3t_bench.json 2> gpurun_out/r3t_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(s1|s2|attn|paged)" -c 200 --csv --log-file gpurun_out/r3t_launches_32k.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/r3t_ncu32.log 2>&1
echo done
