# session 2 call 23: split-KV (KV-range partial prefill + LSE merge) tests, full GPU suite
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "split_kv" > gpurun_out/s2z_tests_split.txt 2>&1; echo "rc=$?" >> gpurun_out/s2z_tests_split.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s2z_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s2z_tests.txt
echo done
