# session 2 call 17: split-K partials through DSMEM (CTA pair) — hang check, parity, A/B
mkdir -p gpurun_out
timeout 60 python tools/s1_timing.py --variant debug --reps 2 > gpurun_out/s2t_dbg.txt 2>&1; echo "rc=$?" >> gpurun_out/s2t_dbg.txt
if grep -q "rc=0" gpurun_out/s2t_dbg.txt; then
  timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s2t_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s2t_tests.txt
  for v in "" nopk "" nopk; do timeout 120 python tools/s1_timing.py --variant "$v" >> gpurun_out/s2t_s1.txt 2>&1; done
  for v in "" nopk; do timeout 120 python tools/s1_timing.py --variant "$v" --d 256 --hq 16 >> gpurun_out/s2t_s1.txt 2>&1; done
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(s1|s2|paged)" -c 40 --csv --log-file gpurun_out/s2t_launches32.csv python tools/s1_timing.py --reps 2 > gpurun_out/s2t_ncu.log 2>&1
  timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/s2t_bench.json 2> gpurun_out/s2t_bench.err
fi
echo done
