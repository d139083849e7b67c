#!/bin/bash
# e2e after moving the per-step energy D2H to the download stream: split vs fused, same box
mkdir -p gpurun_out
export PIF_E2E_TRACE=1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c40_a.json 2> gpurun_out/c40_a.err
PIF_E2E_SPLIT=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c40_c.json 2> gpurun_out/c40_c.err
timeout 600 python tools/e2e_timeline.py 27 16 > gpurun_out/c40_tl.txt 2>&1
timeout 300 python tools/pcie_probe.py > gpurun_out/c40_pcie.txt 2>&1
echo done
