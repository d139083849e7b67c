#!/bin/bash
# microbench A/B: 64^3 / 2^27 at w = 7 and w = 8, weight cache on/off, spread
# XYZ on/off, bank layouts before/after
L=paper_2605_10729_b200
for eps in 1e-6 1e-7; do
  for lib in $L/libpifb200.so $L/lib_prev.so $L/lib_nox.so; do
    for wc in 0 1; do
      echo -n "$(basename $lib) wc=$wc "; PIF_WEIGHT_CACHE=$wc PIF_B200_LIB=$lib python tools/mb_case.py 64 27 $eps 2>/dev/null
    done
  done
done
bash tools/abn.sh 2 $L/lib_prev.so $L/libpifb200.so
