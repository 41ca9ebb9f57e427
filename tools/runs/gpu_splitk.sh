mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/sk_tests.txt 2>&1; echo "exit $?" >> gpurun_out/sk_tests.txt
if grep -q "exit 0" gpurun_out/sk_tests.txt; then
for v in 1 0 1 0; do
  if [ $v = 1 ]; then export BFLA_TC_SPLITS=1; else unset BFLA_TC_SPLITS; fi
  echo "splits_forced_1=$v" >> gpurun_out/sk.txt
  timeout 300 python tools/s1_timing.py --n 32768 >> gpurun_out/sk.txt 2>&1
  timeout 300 python tools/s1_timing.py --n 4096 --hq 16 --d 256 >> gpurun_out/sk.txt 2>&1
  timeout 300 python tools/s1_timing.py --n 32768 --hq 16 --d 256 >> gpurun_out/sk.txt 2>&1
done
unset BFLA_TC_SPLITS
bash tools/runs/gpu_launches.sh sk_llama32k
fi
