# session 3 call 45: sharding modes at world size 1 on the final code (heads / balanced, torchrun launch)
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --shard heads --steps 5 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/r3zq_heads.json 2> gpurun_out/r3zq_heads.err
timeout 900 python bench.py --shard balanced --steps 5 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/r3zq_bal.json 2> gpurun_out/r3zq_bal.err
timeout 900 python bench.py --workload gemma-d256-32k --steps 10 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/r3zq_gemma.json 2> gpurun_out/r3zq_gemma.err
timeout 900 python bench.py --workload qwen32b-64k-paged --steps 10 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/r3zq_qwen.json 2> gpurun_out/r3zq_qwen.err
echo done
