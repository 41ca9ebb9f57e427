mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/all_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/all_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
echo "rc=$?" >> gpurun_out/smoke.txt
