#!/bin/bash
# TMA plane loads (depth 1, 2, 4) vs the cp.async path (PIF_NO_TMA=1), dense and sparse
L=paper_2605_10729_b200
for cfg in "--N 64 --ppm 512" "--N 128 --ppm 64" "--N 256 --ppm 10"; do
  for v in "cp:$L/libpifb200.so:1" "d1:$L/libpifb200.so:0" "d2:$L/lib_d2.so:0" "d4:$L/lib_d4.so:0"; do
    IFS=: read tag lib notma <<< "$v"
    if [ $notma = 1 ]; then export PIF_NO_TMA=1; else unset PIF_NO_TMA; fi
    PIF_B200_LIB=$lib python bench.py $cfg --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg', '$tag', round(d['value']/1e9,3), 'Gps', round(d['ms_per_step'],2), 'ms', {k: round(v,2) for k,v in r['stage_ms'].items() if k in ('interp_push','spread','bin','fields')})"
  done
done
unset PIF_NO_TMA
