# session 3 call 41: K norms forked after the scores (overlapping the split-K reduce) — bench-context A/B vs prev, tests
mkdir -p gpurun_out
for rep in 1 2; do
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --extra-128k 0 > gpurun_out/r3zn_bench_new$rep.json 2>/dev/null
cp paper_2605_12193_b200/libbfla.so /tmp/libbfla_new.so; cp paper_2605_12193_b200/libbfla_prev.so paper_2605_12193_b200/libbfla.so
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --extra-128k 0 > gpurun_out/r3zn_bench_prev$rep.json 2>/dev/null
cp /tmp/libbfla_new.so paper_2605_12193_b200/libbfla.so
done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3zn_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3zn_tests.txt
echo done
