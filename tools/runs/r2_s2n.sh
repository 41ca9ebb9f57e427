# session 2 call 14: ragged fixup grid-stride (tests + varlen launch list), full GPU tests, bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s2n_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s2n_tests.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/s2n_bench.json 2> gpurun_out/s2n_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(s1|s2|paged)" -c 100 --csv --log-file gpurun_out/s2n_launches_varlen.csv python -c "
import sys; sys.path.insert(0,'.'); import torch, bench; torch.cuda.set_device(0); bench.varlen_timing(torch.device('cuda',0), reps=1)" > gpurun_out/s2n_ncuvar.log 2>&1
echo done
