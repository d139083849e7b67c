#!/bin/bash
# merged spread: full GPU suite, sparse bench lines (paper run, 2 per cell), default bench
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c47_tests.txt 2>&1
timeout 600 python bench.py --N 256 --ppm 10 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c47_sparse.json 2> gpurun_out/c47_sparse.err
timeout 600 python bench.py --N 128 --ppm 16 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c47_2pc.json 2> gpurun_out/c47_2pc.err
PIF_SPREAD_MERGE=0 timeout 600 python bench.py --N 128 --ppm 16 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c47_2pc_off.json 2> gpurun_out/c47_2pc_off.err
PIF_SPREAD_MERGE=2 timeout 600 python bench.py --N 128 --ppm 16 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c47_2pc_m2.json 2> gpurun_out/c47_2pc_m2.err
echo done
