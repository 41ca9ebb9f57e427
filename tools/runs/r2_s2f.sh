# session 2 call 6: softmax critical-path variants A/B + fused exchange (mirrors) tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "mirror or peer" > gpurun_out/s2f_tests_mirror.txt 2>&1; echo "rc=$?" >> gpurun_out/s2f_tests_mirror.txt
timeout 60 python tools/attn_time.py --variant bothdbg --reps 2 --dense 1 > gpurun_out/s2f_bothdbg.txt 2>&1; echo "rc=$?" >> gpurun_out/s2f_bothdbg.txt
timeout 120 python tools/attn_time.py --save /tmp/o_prod.pt >> gpurun_out/s2f_ab.jsonl 2>> gpurun_out/s2f_ab.err
if grep -q "rc=0" gpurun_out/s2f_bothdbg.txt; then
for v in sumafter splitp both; do
  timeout 120 python tools/attn_time.py --variant $v --compare /tmp/o_prod.pt >> gpurun_out/s2f_ab.jsonl 2>> gpurun_out/s2f_ab.err; echo "$v rc=$?" >> gpurun_out/s2f_ab.err
done
timeout 120 python tools/attn_time.py --variant both --workload llama8b-128k --reps 5 >> gpurun_out/s2f_ab.jsonl 2>> gpurun_out/s2f_ab.err
timeout 120 python tools/attn_time.py --workload llama8b-128k --reps 5 >> gpurun_out/s2f_ab.jsonl 2>> gpurun_out/s2f_ab.err
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --bfla-variant both > gpurun_out/s2f_tests_both.txt 2>&1; echo "rc=$?" >> gpurun_out/s2f_tests_both.txt
fi
timeout 120 python tools/attn_time.py >> gpurun_out/s2f_ab.jsonl 2>> gpurun_out/s2f_ab.err
echo done
