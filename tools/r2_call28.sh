#!/bin/bash
# ring kernels below their round-1 density thresholds (long segments since
# round 2): default thresholds vs ring everywhere, wide windows, sparse sets
mkdir -p gpurun_out
for c in "128 24 1e-12" "256 24 1e-12" "128 24 1e-9" "256 24 1e-9" "64 20 1e-12" "64 20 1e-15" "128 24 1e-15"; do
  echo -n "default  "; timeout 600 python tools/mb_case.py $c 2>&1 | tail -1
  echo -n "ring-all "; PIF_RING_SPREAD_MIN=0 PIF_RING_GATHER_MIN=0 timeout 600 python tools/mb_case.py $c 2>&1 | tail -1
done > gpurun_out/c28_ring_density.txt
echo done
