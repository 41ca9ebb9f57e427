# session 3 call 17: split-KV planner with one heavy run per head — GPU parity test and one-GPU shard simulation
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "split_kv" > gpurun_out/r3q_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3q_tests.txt
for wl in llama8b-32k llama8b-128k qwen32b-64k-paged; do for sk in 1 0; do
  timeout 900 python tools/shard_sim.py --workload $wl --skew $sk --reps 5 >> gpurun_out/r3q_shard_sim.jsonl 2>> gpurun_out/r3q_shard_sim.err
done; done
echo done
