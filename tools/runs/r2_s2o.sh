# session 2 call 15: sanitizers on the round-2 paths, Q-ring A/B (after split-P), bench with all BASELINE configs
mkdir -p gpurun_out
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t python tools/sanitize_cases.py > gpurun_out/s2o_sanitizer_$t.log 2>&1; echo "rc=$?" >> gpurun_out/s2o_sanitizer_$t.log
done
timeout 120 python tools/attn_time.py --save /tmp/o_prod.pt >> gpurun_out/s2o_ab.jsonl 2>> gpurun_out/s2o_ab.err
for v in qring "" qring; do timeout 120 python tools/attn_time.py --variant "$v" --compare /tmp/o_prod.pt >> gpurun_out/s2o_ab.jsonl 2>> gpurun_out/s2o_ab.err; done
timeout 120 python tools/attn_time.py --variant qring --workload llama8b-128k --reps 5 >> gpurun_out/s2o_ab.jsonl 2>> gpurun_out/s2o_ab.err
timeout 120 python tools/attn_time.py --workload llama8b-128k --reps 5 >> gpurun_out/s2o_ab.jsonl 2>> gpurun_out/s2o_ab.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s2o_bench.json 2> gpurun_out/s2o_bench.err
echo done
