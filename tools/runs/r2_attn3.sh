# attention3 (one Q tile per item, double-buffered S, column-split softmax): debug run first (traps instead of hangs)
mkdir -p gpurun_out
timeout 60 python tools/attn_time.py --variant attn3dbg --reps 2 --dense 0 > gpurun_out/r2_attn3_dbg.txt 2>&1; echo "attn3dbg rc=$?" >> gpurun_out/r2_attn3_dbg.txt
if grep -q "attn3dbg rc=0" gpurun_out/r2_attn3_dbg.txt; then
  timeout 120 python tools/attn_time.py --save /tmp/o_prod.pt >> gpurun_out/r2_attn3.jsonl 2>> gpurun_out/r2_attn3.err
  timeout 60 python tools/attn_time.py --variant attn3 --compare /tmp/o_prod.pt >> gpurun_out/r2_attn3.jsonl 2>> gpurun_out/r2_attn3.err
  timeout 120 python tools/attn_time.py >> gpurun_out/r2_attn3.jsonl 2>> gpurun_out/r2_attn3.err
  timeout 60 python tools/attn_time.py --variant attn3 --compare /tmp/o_prod.pt >> gpurun_out/r2_attn3.jsonl 2>> gpurun_out/r2_attn3.err
  timeout 400 python -m pytest tests/test_gpu_parity.py -x -q --bfla-variant attn3dbg > gpurun_out/r2_attn3_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_attn3_tests.txt
fi
echo done
