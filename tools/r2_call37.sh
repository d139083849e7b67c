#!/bin/bash
# why the bench's e2e differs from the timeline tool: traces inside bench.py
mkdir -p gpurun_out
export PIF_E2E_TRACE=1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c37_a.json 2> gpurun_out/c37_a.err
PIF_WEIGHT_CACHE=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c37_b.json 2> gpurun_out/c37_b.err
PIF_E2E_SPLIT=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c37_c.json 2> gpurun_out/c37_c.err
echo done
