mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tile_128" > gpurun_out/t128_tests.txt 2>&1; echo "exit $?" >> gpurun_out/t128_tests.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t128_all.txt 2>&1; echo "exit $?" >> gpurun_out/t128_all.txt
