#!/bin/bash
# merged perm copy with warp-shared heavy cells: parity, microbench sweep, sparse bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x > gpurun_out/c58_tests.txt 2>&1
timeout 2400 python tools/microbench.py > gpurun_out/c58_microbench.md 2> gpurun_out/c58_microbench.err
PIF_SPREAD_MERGE=0 timeout 2400 python tools/microbench.py > gpurun_out/c58_microbench_nomerge.md 2> gpurun_out/c58_microbench_nomerge.err
timeout 600 python bench.py --N 256 --ppm 10 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c58_sparse.json 2> gpurun_out/c58_sparse.err
echo done
