mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s2_tests.txt 2>&1; echo "exit $?" >> gpurun_out/s2_tests.txt
if grep -q "exit 0" gpurun_out/s2_tests.txt; then
bash tools/runs/gpu_launches.sh s2_llama128k --workload llama8b-128k
bash tools/runs/gpu_launches.sh s2_llama32k
fi
