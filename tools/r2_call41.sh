#!/bin/bash
mkdir -p gpurun_out
for ppm in 512 64; do
  PPM=$ppm PIF_B200_LIB=paper_2605_10729_b200/lib_phase.so timeout 300 python tools/phase_timing.py >> gpurun_out/c41_phase.txt 2>&1
  PPM=$ppm PIF_WEIGHT_CACHE=0 PIF_B200_LIB=paper_2605_10729_b200/lib_phase.so timeout 300 python tools/phase_timing.py >> gpurun_out/c41_phase.txt 2>&1
done
echo done
