# session 2 call 9: ragged fixup per KV head (tests + varlen timing + launch list), attention timeline after split-P
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ragged or varlen or shapes or group_ or mirror" > gpurun_out/s2i_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s2i_tests.txt
timeout 300 python -c "
import sys, json; sys.path.insert(0,'.')
import torch, bench
torch.cuda.set_device(0)
print(json.dumps(bench.varlen_timing(torch.device('cuda',0))))" > gpurun_out/s2i_varlen.json 2> gpurun_out/s2i_varlen.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(s1|s2|paged)" -c 100 --csv --log-file gpurun_out/s2i_launches_varlen.csv python -c "
import sys; sys.path.insert(0,'.'); import torch, bench; torch.cuda.set_device(0); bench.varlen_timing(torch.device('cuda',0), reps=1)" > gpurun_out/s2i_ncuvar.log 2>&1
timeout 120 python tools/attn_trace.py --dense --out gpurun_out/s2i_trace_dense.json > gpurun_out/s2i_trace_dense.txt 2>&1
timeout 120 python tools/attn_trace.py --out gpurun_out/s2i_trace_sparse.json > gpurun_out/s2i_trace_sparse.txt 2>&1
echo done
