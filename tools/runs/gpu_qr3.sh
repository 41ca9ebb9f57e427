mkdir -p gpurun_out
for rep in 1 2; do
BFLA_LIB_VARIANT= timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/qr3_base_$rep.json 2>&1
BFLA_LIB_VARIANT=qr1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/qr3_qr1_$rep.json 2>&1
BFLA_OTMA=0 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/qr3_otma0_$rep.json 2>&1
BFLA_LIB_VARIANT=qr1 BFLA_OTMA=0 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/qr3_qr1otma0_$rep.json 2>&1
done
