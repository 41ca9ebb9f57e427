mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tiny or shapes or paged or dynamic" > gpurun_out/qpf_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/qpf_tests.txt
for rep in 1 2; do for v in "" old; do
BFLA_LIB_VARIANT=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/qpf_${v:-new}_$rep.json 2>&1
done; done
