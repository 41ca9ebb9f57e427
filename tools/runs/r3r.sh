# session 3 call 18: split-KV planner (pieces <= half the per-SM share, a rank's launches on side streams)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "split_kv" > gpurun_out/r3r_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3r_tests.txt
for a in "llama8b-32k 1" "llama8b-32k 0" "llama8b-128k 1" "qwen32b-64k-paged 1"; do set -- $a
  timeout 900 python tools/shard_sim.py --workload $1 --skew $2 --reps 5 >> gpurun_out/r3r_shard_sim.jsonl 2>> gpurun_out/r3r_shard_sim.err
done
echo done
