# session 2 call 10: NVLS multicast exchange test, mirror tests; ncu full of the ragged fixup kernel
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -s -k "mirror or peer" > gpurun_out/s2j_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s2j_tests.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ragged_fixup" -c 1 -o gpurun_out/s2j_fixup python -c "
import sys; sys.path.insert(0,'.'); import torch, bench; torch.cuda.set_device(0); bench.varlen_timing(torch.device('cuda',0), reps=1)" > gpurun_out/s2j_ncu.log 2>&1
echo done
