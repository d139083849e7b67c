#!/bin/bash
# spread knobs: unroll 4 and per-axis weights vs the defaults (unroll 2, XYZ), spread stage
mkdir -p gpurun_out
ab() {
  l=$1; lib=$2; shift 2
  if [ -n "$lib" ]; then export PIF_B200_LIB=$lib; else unset PIF_B200_LIB; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; st=r['stage_ms']
print('$l', '$*', round(d['value']/1e9,3), 'Gps spread', round(st['spread'],3), 'interp', round(st['interp_push'],3), 'sfrac', round(r['spread']['frac'],4))" >> gpurun_out/c60_ab.txt 2>&1
  unset PIF_B200_LIB
}
for rep in 1 2; do
  ab default "" 
  ab unroll4 paper_2605_10729_b200/lib_su4.so
  ab xyz0 paper_2605_10729_b200/lib_sxyz0.so
done
echo done
