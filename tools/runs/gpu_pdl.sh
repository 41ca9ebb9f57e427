mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pdl_tests.txt 2>&1; echo "exit $?" >> gpurun_out/pdl_tests.txt
if grep -q "exit 0" gpurun_out/pdl_tests.txt; then
for rep in 1 2; do
for v in 0 1; do
  echo "BFLA_PDL=$v" >> gpurun_out/pdl.txt
  BFLA_PDL=$v timeout 300 python tools/s1_timing.py --n 32768 >> gpurun_out/pdl.txt 2>&1
  BFLA_PDL=$v timeout 300 python tools/s1_timing.py --n 131072 >> gpurun_out/pdl.txt 2>&1
  BFLA_PDL=$v timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/pdl_b.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/pdl_b.json'));print('bench', round(d['value'],4), {k: round(v,4) for k,v in d['stages_ms'].items()})" >> gpurun_out/pdl.txt
done
done
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_cases.py > gpurun_out/pdl_synccheck.log 2>&1; echo "exit=$?" >> gpurun_out/pdl_synccheck.log
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_cases.py > gpurun_out/pdl_memcheck.log 2>&1; echo "exit=$?" >> gpurun_out/pdl_memcheck.log
fi
