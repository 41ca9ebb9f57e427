# round 2 session 2, call 1: GPU tests, default bench line, smoke, attention A/B (product / attn3 / split), launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/s2a_gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=20 > gpurun_out/s2a_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s2a_tests.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/s2a_bench.json 2> gpurun_out/s2a_bench.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2a_smoke.txt 2>&1
timeout 60 python tools/attn_time.py --variant attn3dbg --reps 2 --dense 0 > gpurun_out/s2a_attn3dbg.txt 2>&1; echo "rc=$?" >> gpurun_out/s2a_attn3dbg.txt
timeout 120 python tools/attn_time.py --save /tmp/o_prod.pt >> gpurun_out/s2a_ab.jsonl 2>> gpurun_out/s2a_ab.err
if grep -q "rc=0" gpurun_out/s2a_attn3dbg.txt; then
timeout 120 python tools/attn_time.py --variant attn3 --compare /tmp/o_prod.pt >> gpurun_out/s2a_ab.jsonl 2>> gpurun_out/s2a_ab.err
fi
timeout 120 python tools/attn_time.py --variant split --compare /tmp/o_prod.pt >> gpurun_out/s2a_ab.jsonl 2>> gpurun_out/s2a_ab.err
timeout 120 python tools/attn_time.py >> gpurun_out/s2a_ab.jsonl 2>> gpurun_out/s2a_ab.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s2a_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/s2a_ncu_bench.log 2>&1
echo done
