#!/bin/bash
# e2e timeline breakdown: default, PIF_PUSH_AGG=0 (no per-load check), scatter-after-push
mkdir -p gpurun_out
timeout 600 python tools/e2e_timeline.py 27 16 > gpurun_out/c31_tl_default.txt 2>&1
PIF_PUSH_AGG=0 timeout 600 python tools/e2e_timeline.py 27 16 > gpurun_out/c31_tl_noagg.txt 2>&1
PIF_E2E_SCATTER=1 timeout 600 python tools/e2e_timeline.py 27 16 > gpurun_out/c31_tl_scatter.txt 2>&1
timeout 600 python tools/e2e_timeline.py 27 4 > gpurun_out/c31_tl_4chunks.txt 2>&1
echo done
