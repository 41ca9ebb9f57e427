# what-if timing of the softmax phases of k_attn2 (A/B builds; results invalid by design except product/poly)
mkdir -p gpurun_out
for v in "" noload nostore nols noexp poly0 poly55 ""; do
  timeout 300 python tools/attn_time.py --variant "$v" >> gpurun_out/r2_whatif.jsonl 2>> gpurun_out/r2_whatif.err
done
echo done
