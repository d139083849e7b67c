#!/bin/bash
# round-2 knob sweep on one box: gather FMA-tail threshold (libraries) and the
# work-item size (PIF_SEG_TARGET), default bench workload
L=paper_2605_10729_b200
bash tools/abn.sh 2 $L/libpifb200.so $L/lib_fma2.so $L/lib_fma4.so $L/lib_fma5.so
bash tools/envsweep.sh "--steps 10 --warmup 3" PIF_SEG_TARGET 512 768 1024
