#!/bin/bash
# e2e with 32 hardware queues: split vs fused, traces inside bench.py
mkdir -p gpurun_out
export PIF_E2E_TRACE=1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c38_a.json 2> gpurun_out/c38_a.err
PIF_E2E_SPLIT=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c38_c.json 2> gpurun_out/c38_c.err
CUDA_DEVICE_MAX_CONNECTIONS=8 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c38_d.json 2> gpurun_out/c38_d.err
echo done
