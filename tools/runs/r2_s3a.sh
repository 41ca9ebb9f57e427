# session 2 call 24: FMA-pipe exp2 fraction re-tuned after split-PV issue (0, 1/8, 1/4 (current), 3/8)
mkdir -p gpurun_out
timeout 120 python tools/attn_time.py --save /tmp/o_prod.pt >> gpurun_out/s3a_ab.jsonl 2>> gpurun_out/s3a_ab.err
for v in p00 p02 "" p26 p00 p02 "" p26; do timeout 120 python tools/attn_time.py --variant "$v" --compare /tmp/o_prod.pt >> gpurun_out/s3a_ab.jsonl 2>> gpurun_out/s3a_ab.err; done
for v in p00 p02 "" p26; do timeout 120 python tools/attn_time.py --variant "$v" --workload llama8b-128k --reps 5 >> gpurun_out/s3a_ab.jsonl 2>> gpurun_out/s3a_ab.err; done
echo done
