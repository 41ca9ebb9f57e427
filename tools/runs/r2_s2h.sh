# session 2 call 8: split-P default — full GPU tests, smoke, bench, launch lists (32K, 128K, varlen), mirror cost
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s2h_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s2h_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2h_smoke.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/s2h_bench.json 2> gpurun_out/s2h_bench.err
timeout 300 python tools/mirror_time.py > gpurun_out/s2h_mirror.jsonl 2>&1
timeout 300 python tools/mirror_time.py --workload llama8b-128k --reps 3 >> gpurun_out/s2h_mirror.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(s1|s2|attn|paged)" -c 200 --csv --log-file gpurun_out/s2h_launches_32k.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/s2h_ncu32.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(s1|s2|paged)" -c 100 --csv --log-file gpurun_out/s2h_launches_128k.csv python bench.py --workload llama8b-128k --steps 2 --warmup 3 --no-cpu-baseline --extra-128k 0 > gpurun_out/s2h_ncu128.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(s1|s2|attn|paged)" -c 100 --csv --log-file gpurun_out/s2h_launches_varlen.csv python -c "
import sys; sys.path.insert(0,'.'); import torch, bench; torch.cuda.set_device(0); bench.varlen_timing(torch.device('cuda',0), reps=1)" > gpurun_out/s2h_ncuvar.log 2>&1
echo done
