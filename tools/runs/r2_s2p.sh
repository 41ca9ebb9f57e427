# session 2 call 16: two query heads per Stage-1 score CTA (default) — hang check, parity, A/B vs one head
mkdir -p gpurun_out
timeout 60 python tools/s1_timing.py --variant debug --reps 2 > gpurun_out/s2r_dbg.txt 2>&1; echo "rc=$?" >> gpurun_out/s2r_dbg.txt
if grep -q "rc=0" gpurun_out/s2r_dbg.txt; then
  timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s2r_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s2r_tests.txt
  for v in "" h1 "" h1; do timeout 120 python tools/s1_timing.py --variant "$v" >> gpurun_out/s2r_s1.txt 2>&1; done
  for v in "" h1 ""; do timeout 120 python tools/s1_timing.py --variant "$v" --n 131072 --reps 5 >> gpurun_out/s2r_s1.txt 2>&1; done
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(s1|s2|paged)" -c 40 --csv --log-file gpurun_out/s2r_launches128.csv python tools/s1_timing.py --n 131072 --reps 2 > gpurun_out/s2r_ncu.log 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(s1|s2|paged)" -c 40 --csv --log-file gpurun_out/s2r_launches32.csv python tools/s1_timing.py --reps 2 >> gpurun_out/s2r_ncu.log 2>&1
fi
echo done
