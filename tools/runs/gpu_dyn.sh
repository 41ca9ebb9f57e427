mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/dyn_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/dyn_tests.txt
if grep -q "rc=0" gpurun_out/dyn_tests.txt; then
for rep in 1 2; do for v in 1 0; do
BFLA_DYN_SCHED=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/dyn_${v}_$rep.json 2>&1
done; done
BFLA_DYN_SCHED=1 timeout 300 python bench.py --workload llama8b-128k --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/dyn_1_128k.json 2>&1
BFLA_DYN_SCHED=0 timeout 300 python bench.py --workload llama8b-128k --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/dyn_0_128k.json 2>&1
fi
