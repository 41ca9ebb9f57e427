# session 3 call 29: key-group norms from the score kernel's B stages (no k_s1_block_norms): norms check, A/B, GPU suite, bench
mkdir -p gpurun_out
timeout 600 python tools/norm_check.py > gpurun_out/r3zc_norms.txt 2>&1
for rep in 1 2; do for n in 32768 131072 65536 8192; do
  BFLA_S1_KNORM_KERNEL=1 timeout 300 python tools/s1_timing.py --n $n --variant exp >> gpurun_out/r3zc_s1.txt 2>&1
  timeout 300 python tools/s1_timing.py --n $n >> gpurun_out/r3zc_s1.txt 2>&1
done; done
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r3zc_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3zc_tests.txt
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r3zc_bench.json 2> gpurun_out/r3zc_bench.err
echo done
