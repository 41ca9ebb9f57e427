# session 2 call 13: CTA-pair (cta_group::2) Stage-1 scores A/B — hang check, parity, timing
mkdir -p gpurun_out
timeout 60 python tools/s1_timing.py --variant pairdbg --reps 2 > gpurun_out/s2m_pairdbg.txt 2>&1; echo "rc=$?" >> gpurun_out/s2m_pairdbg.txt
if grep -q "rc=0" gpurun_out/s2m_pairdbg.txt; then
  timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --bfla-variant pair > gpurun_out/s2m_tests_pair.txt 2>&1; echo "rc=$?" >> gpurun_out/s2m_tests_pair.txt
  timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q --bfla-variant pair > gpurun_out/s2m_tests_full_pair.txt 2>&1; echo "rc=$?" >> gpurun_out/s2m_tests_full_pair.txt
  for v in "" pair "" pair; do timeout 120 python tools/s1_timing.py --variant "$v" >> gpurun_out/s2m_s1.txt 2>&1; done
  for v in "" pair; do timeout 120 python tools/s1_timing.py --variant "$v" --n 131072 --reps 5 >> gpurun_out/s2m_s1.txt 2>&1; done
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(s1|s2|paged)" -c 40 --csv --log-file gpurun_out/s2m_launches_pair128.csv python tools/s1_timing.py --variant pair --n 131072 --reps 2 > gpurun_out/s2m_ncu.log 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(s1|s2|paged)" -c 40 --csv --log-file gpurun_out/s2m_launches_pair32.csv python tools/s1_timing.py --variant pair --reps 2 >> gpurun_out/s2m_ncu.log 2>&1
fi
echo done
