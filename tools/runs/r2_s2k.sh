# session 2 call 11: Q tiles shared by both softmax warpgroups (SMX=3) A/B + parity
mkdir -p gpurun_out
timeout 60 python tools/attn_time.py --variant shareddbg --reps 2 --dense 1 > gpurun_out/s2k_shareddbg.txt 2>&1; echo "rc=$?" >> gpurun_out/s2k_shareddbg.txt
timeout 120 python tools/attn_time.py --save /tmp/o_prod.pt >> gpurun_out/s2k_ab.jsonl 2>> gpurun_out/s2k_ab.err
if grep -q "rc=0" gpurun_out/s2k_shareddbg.txt; then
  timeout 120 python tools/attn_time.py --variant shared --compare /tmp/o_prod.pt >> gpurun_out/s2k_ab.jsonl 2>> gpurun_out/s2k_ab.err
  timeout 120 python tools/attn_time.py --variant shared --workload llama8b-128k --reps 5 >> gpurun_out/s2k_ab.jsonl 2>> gpurun_out/s2k_ab.err
  timeout 120 python tools/attn_time.py --workload llama8b-128k --reps 5 >> gpurun_out/s2k_ab.jsonl 2>> gpurun_out/s2k_ab.err
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --bfla-variant shared > gpurun_out/s2k_tests_shared.txt 2>&1; echo "rc=$?" >> gpurun_out/s2k_tests_shared.txt
  timeout 120 python tools/attn_time.py --variant shared --compare /tmp/o_prod.pt >> gpurun_out/s2k_ab.jsonl 2>> gpurun_out/s2k_ab.err
fi
timeout 120 python tools/attn_time.py >> gpurun_out/s2k_ab.jsonl 2>> gpurun_out/s2k_ab.err
echo done
