mkdir -p gpurun_out
BFLA_LIB_VARIANT=kv timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "shapes or tiny_structured or dynamic" > gpurun_out/kvs_tests.txt 2>&1; echo "exit $?" >> gpurun_out/kvs_tests.txt
for rep in 1 2; do
for v in base kv; do
  if [ $v = kv ]; then export BFLA_LIB_VARIANT=kv; else unset BFLA_LIB_VARIANT; fi
  for wl in llama8b-32k llama8b-128k; do
    timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/kvs_b.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/kvs_b.json'));print('$v $wl', round(d['value'],4), 'attn', round(d['stages_ms']['sparse_prefill'],4), 'dense', round(d['dense_ms'],3), d['clocks']['sm_mhz'])" >> gpurun_out/kvs.txt
  done
done
done
