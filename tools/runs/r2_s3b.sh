# session 2 call 25: split-KV on a row slice, POLY 1/8 default — full GPU suite, smoke, bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s3b_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s3b_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3b_smoke.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s3b_bench.json 2> gpurun_out/s3b_bench.err
echo done
