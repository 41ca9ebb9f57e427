# session 2 call 21: torchrun-launched KV-head-sharded bench at world 1 (stdout flushed), epilogue A/B
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr=127.0.0.1 --master-port=29513 bench.py --gpus 1 --shard heads --workload llama8b-32k --steps 5 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/s2x_heads_auto.json 2> gpurun_out/s2x_heads_auto.err; echo "rc=$?" >> gpurun_out/s2x_heads_auto.err
timeout 120 python tools/attn_time.py --save /tmp/o_prod.pt >> gpurun_out/s2x_ab.jsonl 2>> gpurun_out/s2x_ab.err
for v in epi "" epi; do timeout 120 python tools/attn_time.py --variant "$v" --compare /tmp/o_prod.pt >> gpurun_out/s2x_ab.jsonl 2>> gpurun_out/s2x_ab.err; done
for v in epi ""; do timeout 120 python tools/attn_time.py --variant "$v" --workload llama8b-128k --reps 5 >> gpurun_out/s2x_ab.jsonl 2>> gpurun_out/s2x_ab.err; done
echo done
