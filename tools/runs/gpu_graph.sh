mkdir -p gpurun_out
for g in 0 1 0 1; do
timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --graph $g > gpurun_out/graph_$g.json 2>gpurun_out/graph_$g.err
python -c "import json;d=json.load(open('gpurun_out/graph_$g.json'));print('graph=$g', round(d['value'],4), d['stages_ms'], d['gpu_launches'], d['launch'], d['e2e']['value'])" >> gpurun_out/graph.txt
done
