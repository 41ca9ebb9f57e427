# A/B: softmax ping-pong variants vs product, same box
mkdir -p gpurun_out
for v in "" pp1 pp2 "" pp1 pp2; do
  timeout 300 python tools/attn_time.py --variant "$v" >> gpurun_out/r2_pp.jsonl 2>> gpurun_out/r2_pp.err
done
echo done
