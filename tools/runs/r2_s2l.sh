# session 2 call 12: staged ragged fixup (tests + varlen timing + launch list)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ragged or varlen or shapes or group_ or mirror or peer" > gpurun_out/s2l_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s2l_tests.txt
timeout 300 python -c "
import sys, json; sys.path.insert(0,'.')
import torch, bench
torch.cuda.set_device(0)
print(json.dumps(bench.varlen_timing(torch.device('cuda',0))))" > gpurun_out/s2l_varlen.json 2> gpurun_out/s2l_varlen.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(s1|s2|paged)" -c 100 --csv --log-file gpurun_out/s2l_launches_varlen.csv python -c "
import sys; sys.path.insert(0,'.'); import torch, bench; torch.cuda.set_device(0); bench.varlen_timing(torch.device('cuda',0), reps=1)" > gpurun_out/s2l_ncuvar.log 2>&1
echo done
