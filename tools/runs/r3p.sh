# session 3 call 16: split-KV planner — GPU parity test and the one-GPU shard simulation (diffuse head)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "split_kv" > gpurun_out/r3p_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3p_tests.txt
for wl in llama8b-32k llama8b-128k; do for sk in 0 1; do
  timeout 900 python tools/shard_sim.py --workload $wl --skew $sk --reps 5 >> gpurun_out/r3p_shard_sim.jsonl 2>> gpurun_out/r3p_shard_sim.err
done; done
echo done
