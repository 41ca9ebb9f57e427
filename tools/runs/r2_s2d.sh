# session 2 call 4: ragged fixup (partial pairs) tests + varlen bench point; attention what-if sensitivities
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ragged or varlen or group_ or shapes" > gpurun_out/s2d_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s2d_tests.txt
timeout 300 python -c "
import sys, json; sys.argv=['bench']; sys.path.insert(0,'.')
import torch, bench
torch.cuda.set_device(0)
print(json.dumps(bench.varlen_timing(torch.device('cuda',0))))" > gpurun_out/s2d_varlen.json 2> gpurun_out/s2d_varlen.err
timeout 120 python tools/attn_time.py --save /tmp/o_prod.pt >> gpurun_out/s2d_ab.jsonl 2>> gpurun_out/s2d_ab.err
for v in noexp nostore noload poly0 polyall poly8; do
  timeout 120 python tools/attn_time.py --variant $v --compare /tmp/o_prod.pt >> gpurun_out/s2d_ab.jsonl 2>> gpurun_out/s2d_ab.err; echo "$v rc=$?" >> gpurun_out/s2d_ab.err
done
timeout 60 python tools/attn_time.py --variant splitdbg --reps 2 --dense 0 > gpurun_out/s2d_splitdbg.txt 2>&1; echo "rc=$?" >> gpurun_out/s2d_splitdbg.txt
timeout 120 python tools/attn_time.py >> gpurun_out/s2d_ab.jsonl 2>> gpurun_out/s2d_ab.err
echo done
