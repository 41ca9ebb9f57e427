mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "head_dim or varlen or tiny_structured" > gpurun_out/dyn1_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/dyn1_tests.txt
BFLA_ATTN=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/dyn1_tests_v1.txt 2>&1
echo "rc=$?" >> gpurun_out/dyn1_tests_v1.txt
for v in 1 0; do
BFLA_DYN_SCHED=$v timeout 300 python bench.py --workload gemma-d256-32k --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/dyn1_gemma_$v.json 2>&1
done
