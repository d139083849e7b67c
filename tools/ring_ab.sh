#!/bin/bash
# ring kernels (w = 13) with long items vs the previous build, microbench cases
L=paper_2605_10729_b200
for c in "64 24 1e-12" "32 24 1e-12" "128 24 1e-12" "64 24 1e-9"; do
  for lib in $L/lib_prev.so $L/libpifb200.so; do
    echo -n "$(basename $lib) "; PIF_B200_LIB=$lib python tools/mb_case.py $c 2>/dev/null
  done
done
