# usage: bash tools/runs/gpu_launches.sh TAG [bench args...]  -> gpurun_out/launches_TAG.csv (one bench step)
mkdir -p gpurun_out
tag=$1; shift
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_s1|k_s2|k_attn|k_paged" -c 60 --csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline "$@" > gpurun_out/launches_$tag.csv 2>&1
