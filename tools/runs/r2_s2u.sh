# session 2 call 18: O epilogue through per-thread global stores (Q slot freed by the last S MMA) vs TMA store
mkdir -p gpurun_out
timeout 120 python tools/attn_time.py --save /tmp/o_prod.pt >> gpurun_out/s2u_ab.jsonl 2>> gpurun_out/s2u_ab.err
for i in 1 2; do
  BFLA_OTMA=0 timeout 120 python tools/attn_time.py --variant exp --compare /tmp/o_prod.pt >> gpurun_out/s2u_ab.jsonl 2>> gpurun_out/s2u_ab.err
  timeout 120 python tools/attn_time.py --variant exp --compare /tmp/o_prod.pt >> gpurun_out/s2u_ab.jsonl 2>> gpurun_out/s2u_ab.err
done
BFLA_OTMA=0 timeout 120 python tools/attn_time.py --variant exp --workload llama8b-128k --reps 5 >> gpurun_out/s2u_ab.jsonl 2>> gpurun_out/s2u_ab.err
timeout 120 python tools/attn_time.py --variant exp --workload llama8b-128k --reps 5 >> gpurun_out/s2u_ab.jsonl 2>> gpurun_out/s2u_ab.err
echo done
