mkdir -p gpurun_out
BFLA_ATTN=4 timeout 240 python -m pytest tests/test_gpu_parity.py -x -q -k "tiny_structured or test_shapes or dense_matches or keep_all" > gpurun_out/a4_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/a4_tests.txt
if grep -q "rc=0" gpurun_out/a4_tests.txt; then
BFLA_ATTN=4 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "paged or varlen or strided or per_query" >> gpurun_out/a4_tests.txt 2>&1
echo "rc2=$?" >> gpurun_out/a4_tests.txt
for v in 2 4; do BFLA_ATTN=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/a4_bench_$v.json 2>&1; done
fi
