mkdir -p gpurun_out
timeout 120 python tools/attn_time.py --save /tmp/o_prod.pt >> gpurun_out/r2_split4.jsonl 2>> gpurun_out/r2_split4.err
for v in splitA splitB splitC; do
timeout 40 python tools/attn_time.py --variant $v --compare /tmp/o_prod.pt >> gpurun_out/r2_split4.jsonl 2>> gpurun_out/r2_split4.err; echo "$v rc=$?" >> gpurun_out/r2_split4.err
done
echo done
