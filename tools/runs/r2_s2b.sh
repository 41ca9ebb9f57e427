# session 2 call 2: f1 ragged/varlen tensor-core Stage 1 + f3 G=16 / g=1 tests, Tab.mask sweep, launch list (our kernels)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ragged or varlen or group_ or shapes" > gpurun_out/s2b_tests_new.txt 2>&1; echo "rc=$?" >> gpurun_out/s2b_tests_new.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s2b_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s2b_tests.txt
timeout 600 python tools/mask_sweep.py --out gpurun_out/s2b_tabmask_sweep.md > gpurun_out/s2b_sweep.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(s1|s2|attn|paged)" -c 200 --csv --log-file gpurun_out/s2b_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/s2b_ncu_bench.log 2>&1
echo done
