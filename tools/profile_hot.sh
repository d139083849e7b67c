#!/bin/bash
# ncu --set full (with source counters) of the two hot kernels in steady state at
# the bench config, plus the launch list.  Outputs under gpurun_out/ (tag = $1).
tag=${1:-r2}
shift
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-e2e \
    --no-cpu-baseline "$@" > gpurun_out/ncu_l_$tag.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"spread_mma|interp_mma" -s 4 -c 2 \
    -f -o gpurun_out/prof_$tag python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
    "$@" > gpurun_out/ncu_f_$tag.log 2>&1
echo "profile $tag done"
