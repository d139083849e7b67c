#!/bin/bash
# TMA plane loads vs the cp.async path (PIF_NO_TMA=1), dense and sparse
for cfg in "--N 64 --ppm 512" "--N 128 --ppm 64" "--N 256 --ppm 10"; do
  for t in 0 1; do
    if [ $t = 1 ]; then export PIF_NO_TMA=1; else unset PIF_NO_TMA; fi
    python bench.py $cfg --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg', 'no_tma=$t', round(d['value']/1e9,3), 'Gps', round(d['ms_per_step'],2), 'ms', {k: round(v,2) for k,v in r['stage_ms'].items() if k in ('interp_push','spread','bin','fields')})"
  done
done
unset PIF_NO_TMA
