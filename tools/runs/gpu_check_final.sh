mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/final_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.txt 2>&1
timeout 600 python bench.py --steps 30 --warmup 3 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
