# session 3 call 3: debug the certification norms of the Gram-free scores kernel
mkdir -p gpurun_out
timeout 600 python tools/norm_check.py > gpurun_out/r3c_norms.txt 2>&1
echo done
