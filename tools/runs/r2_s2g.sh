# session 2 call 7: split-P variants (1/2 split, 1/2 with hidden wait, 3/4 split with hidden wait)
mkdir -p gpurun_out
for v in splitp2dbg splitp3dbg; do
timeout 60 python tools/attn_time.py --variant $v --reps 2 --dense 1 > gpurun_out/s2g_$v.txt 2>&1; echo "rc=$?" >> gpurun_out/s2g_$v.txt
done
timeout 120 python tools/attn_time.py --save /tmp/o_prod.pt >> gpurun_out/s2g_ab.jsonl 2>> gpurun_out/s2g_ab.err
for v in splitp splitp2 splitp3 splitp splitp2 splitp3; do
  timeout 120 python tools/attn_time.py --variant $v --compare /tmp/o_prod.pt >> gpurun_out/s2g_ab.jsonl 2>> gpurun_out/s2g_ab.err; echo "$v rc=$?" >> gpurun_out/s2g_ab.err
done
for v in splitp splitp2 splitp3; do
  timeout 120 python tools/attn_time.py --variant $v --workload llama8b-128k --reps 5 >> gpurun_out/s2g_ab.jsonl 2>> gpurun_out/s2g_ab.err
done
timeout 120 python tools/attn_time.py --workload llama8b-128k --reps 5 >> gpurun_out/s2g_ab.jsonl 2>> gpurun_out/s2g_ab.err
timeout 120 python tools/attn_time.py >> gpurun_out/s2g_ab.jsonl 2>> gpurun_out/s2g_ab.err
echo done
