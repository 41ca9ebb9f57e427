# session 2 call 19: KV-head-sharded bench path under torchrun (world 1): fused exchange + self-check, NCCL path
mkdir -p gpurun_out
for ex in auto nccl; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr=127.0.0.1 --master-port=29511 bench.py --gpus 1 --shard heads --exchange $ex --workload llama8b-32k --steps 5 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/s2v_heads_$ex.json 2> gpurun_out/s2v_heads_$ex.err
done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s2v_bench.json 2> gpurun_out/s2v_bench.err
echo done
