# round 2 check 1: build, GPU tests (incl. new full-size cases), bench default line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2c1_build.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r2c1_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2c1_tests.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2c1_bench.json 2> gpurun_out/r2c1_bench.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c1_smoke.txt 2>&1
echo done
