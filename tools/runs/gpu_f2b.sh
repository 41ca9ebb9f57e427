mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f2_tests.txt 2>&1
echo "tests exit $?" >> gpurun_out/f2_tests.txt
for sk in 0 1; do
for wl in llama8b-32k llama8b-128k qwen32b-64k-paged; do
  timeout 400 python tools/shard_sim.py --workload $wl --skew $sk >> gpurun_out/f2_shard_sim.jsonl 2>> gpurun_out/f2_shard_sim.err
done
done
