# A/B: column-split softmax (two warpgroups per Q tile) vs product; O compared on a sample; parity tests on the variant
mkdir -p gpurun_out
timeout 300 python tools/attn_time.py --save /tmp/o_prod.pt >> gpurun_out/r2_split.jsonl 2>> gpurun_out/r2_split.err
timeout 300 python tools/attn_time.py --variant split --compare /tmp/o_prod.pt >> gpurun_out/r2_split.jsonl 2>> gpurun_out/r2_split.err
timeout 300 python tools/attn_time.py >> gpurun_out/r2_split.jsonl 2>> gpurun_out/r2_split.err
timeout 300 python tools/attn_time.py --variant split --compare /tmp/o_prod.pt >> gpurun_out/r2_split.jsonl 2>> gpurun_out/r2_split.err
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --bfla-variant split > gpurun_out/r2_split_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_split_tests.txt
echo done
