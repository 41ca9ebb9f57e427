mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/kc_tests.txt 2>&1; echo "exit $?" >> gpurun_out/kc_tests.txt
if grep -q "exit 0" gpurun_out/kc_tests.txt; then
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_cases.py > gpurun_out/kc_memcheck.log 2>&1; echo "exit=$?" >> gpurun_out/kc_memcheck.log
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_cases.py > gpurun_out/kc_racecheck.log 2>&1; echo "exit=$?" >> gpurun_out/kc_racecheck.log
for v in 2 0 2 0; do
  echo "BFLA_RECOMPUTE=$v" >> gpurun_out/kc.txt
  BFLA_RECOMPUTE=$v timeout 300 python tools/s1_timing.py --n 32768 --hq 16 --d 256 >> gpurun_out/kc.txt 2>&1
  BFLA_RECOMPUTE=$v timeout 300 python tools/s1_timing.py --n 131072 --hq 16 --d 256 >> gpurun_out/kc.txt 2>&1
  BFLA_RECOMPUTE=$v timeout 300 python tools/s1_timing.py --n 131072 --hq 16 --d 256 --ratio 0.1 >> gpurun_out/kc.txt 2>&1
done
fi
