mkdir -p gpurun_out
for g in 1 0 1 0; do
timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --graph $g > gpurun_out/graph_$g.json 2>gpurun_out/graph_$g.err
python -c "import json;d=json.load(open('gpurun_out/graph_$g.json'));print('graph=$g', round(d['value'],4), {k: round(v,4) for k,v in d['stages_ms'].items()}, round(d['roofline']['frac'],3), d['gpu_launches'])" >> gpurun_out/graph2.txt
done
