# session 3 call 27: full GPU suite, smoke, bench line after the K-norm launch-order change
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r3za_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3za_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3za_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r3za_smoke.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r3za_bench.json 2> gpurun_out/r3za_bench.err
echo done
