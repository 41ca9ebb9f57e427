# session 2 call 20: debug the KV-head-sharded bench path at world 1 (no torchrun wrapper)
mkdir -p gpurun_out
for ex in nccl auto; do
  RANK=0 WORLD_SIZE=1 LOCAL_RANK=0 MASTER_ADDR=127.0.0.1 MASTER_PORT=29512 timeout 600 python -X faulthandler bench.py --gpus 1 --shard heads --exchange $ex --workload llama8b-32k --steps 5 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/s2w_heads_$ex.json 2> gpurun_out/s2w_heads_$ex.err; echo "rc=$?" >> gpurun_out/s2w_heads_$ex.err
done
echo done
