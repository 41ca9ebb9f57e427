mkdir -p gpurun_out
for rep in 1 2 3; do
  for v in old new; do
    if [ $v = old ]; then export BFLA_LIB_VARIANT=old; else unset BFLA_LIB_VARIANT; fi
    timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/abf2_tmp.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/abf2_tmp.json'));print('$v', round(d['ms_per_step'],4), 'attn', round(d['stages_ms']['sparse_prefill'],4), 's1', round(d['stages_ms']['stage1_scores_select'],4), d['clocks']['sm_mhz'])" >> gpurun_out/abf2.txt
  done
done
