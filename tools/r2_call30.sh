#!/bin/bash
# HEAD: full GPU suite, e2e timeline (id-order host set put into cell order once
# per step), default bench line, Penning line, ncu of the hot kernels.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/c30_tests.txt 2>&1
timeout 600 python tools/e2e_timeline.py 27 16 > gpurun_out/c30_e2e_timeline.txt 2>&1
timeout 900 python bench.py > gpurun_out/c30_bench.json 2> gpurun_out/c30_bench.err
timeout 600 python bench.py --kind penning --no-cpu-baseline > gpurun_out/c30_penning.json 2> /dev/null
bash tools/profile_hot.sh c30
python tools/ncu_summary.py full gpurun_out/prof_c30.ncu-rep > gpurun_out/c30_full.md 2>&1
python tools/ncu_summary.py launches gpurun_out/launches_c30.csv > gpurun_out/c30_launches.md 2>&1
echo done
