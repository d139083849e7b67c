#!/bin/bash
# source-level (SASS) stall attribution of the spread and the gather at the bench config
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:"spread_mma|interp_mma" -s 4 -c 2 \
    -f -o gpurun_out/prof_c43 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c43.log 2>&1
ncu -i gpurun_out/prof_c43.ncu-rep --page source --csv --print-source sass -k regex:spread_mma > gpurun_out/c43_spread_sass.csv 2>&1
ncu -i gpurun_out/prof_c43.ncu-rep --page source --csv --print-source sass -k regex:interp_mma > gpurun_out/c43_interp_sass.csv 2>&1
python tools/ncu_sass_stalls.py gpurun_out/c43_spread_sass.csv > gpurun_out/c43_spread_stalls.txt 2>&1
python tools/ncu_sass_stalls.py gpurun_out/c43_interp_sass.csv > gpurun_out/c43_interp_stalls.txt 2>&1
ls -la gpurun_out/
echo done
