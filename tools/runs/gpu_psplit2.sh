mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/ps_tests.txt 2>&1; echo "exit $?" >> gpurun_out/ps_tests.txt
if grep -q "exit 0" gpurun_out/ps_tests.txt; then
for wl in llama8b-32k llama8b-128k; do
for rep in 1 2; do
  for v in old new; do
    if [ $v = old ]; then export BFLA_LIB_VARIANT=old; else unset BFLA_LIB_VARIANT; fi
    timeout 300 python bench.py --workload $wl --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ps_tmp.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ps_tmp.json'));print('$wl $v', round(d['ms_per_step'],4), 'attn', round(d['stages_ms']['sparse_prefill'],4), 'dense', round(d['dense_ms'],3), d['clocks']['sm_mhz'])" >> gpurun_out/ps.txt
  done
done
done
fi
