# A/B: split softmax with register slack (56/112); short timeouts; then Stage-1 in-kernel split-K reduce check
mkdir -p gpurun_out
timeout 120 python tools/attn_time.py --save /tmp/o_prod.pt >> gpurun_out/r2_split2.jsonl 2>> gpurun_out/r2_split2.err
timeout 60 python tools/attn_time.py --variant split2 --compare /tmp/o_prod.pt >> gpurun_out/r2_split2.jsonl 2>> gpurun_out/r2_split2.err
echo "split2 rc=$?" >> gpurun_out/r2_split2.err
timeout 60 python tools/attn_time.py --variant split2dbg --reps 2 --dense 0 >> gpurun_out/r2_split2.jsonl 2>> gpurun_out/r2_split2.err
echo "split2dbg rc=$?" >> gpurun_out/r2_split2.err
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "fast_scores or certification_norms or keep_ratio or chunked or graph or deterministic" > gpurun_out/r2_s1_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_s1_tests.txt
timeout 120 python tools/s1_timing.py > gpurun_out/r2_s1_timing.txt 2>&1
timeout 120 python tools/s1_timing.py --n 131072 >> gpurun_out/r2_s1_timing.txt 2>&1
echo done
