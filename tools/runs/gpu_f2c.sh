mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "balanced or row_slices" > gpurun_out/f2c_tests.txt 2>&1
echo "tests exit $?" >> gpurun_out/f2c_tests.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --shard balanced --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/f2c_bench_bal.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/f2c_bench.txt 2>&1
