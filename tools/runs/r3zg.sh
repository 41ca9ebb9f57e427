# session 3 call 33: CTA-pair (cta_group::2) score kernel — debug build first (mbarrier traps), then parity + A/B
mkdir -p gpurun_out
for n in 8192 32768; do timeout 120 python tools/s1_timing.py --n $n --variant dbg --reps 3 >> gpurun_out/r3zg_dbg.txt 2>&1; echo "rc=$?" >> gpurun_out/r3zg_dbg.txt; done
if grep -q "rc=0" gpurun_out/r3zg_dbg.txt && ! grep -q "rc=[1-9]" gpurun_out/r3zg_dbg.txt; then
  timeout 300 python tools/norm_check.py > gpurun_out/r3zg_norms.txt 2>&1
  for rep in 1 2; do for n in 32768 131072 8192; do
    BFLA_S1_PAIR=0 timeout 120 python tools/s1_timing.py --n $n --variant exp >> gpurun_out/r3zg_s1.txt 2>&1
    timeout 120 python tools/s1_timing.py --n $n >> gpurun_out/r3zg_s1.txt 2>&1
  done; done
  timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3zg_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r3zg_tests.txt
fi
echo done
