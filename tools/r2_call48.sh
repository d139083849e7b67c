#!/bin/bash
mkdir -p gpurun_out
for ppm in 10 64; do
  PPM=$ppm PIF_B200_LIB=paper_2605_10729_b200/lib_phase.so timeout 300 python tools/phase_timing.py >> gpurun_out/c48_phase.txt 2>&1
done
echo done
