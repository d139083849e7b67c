#!/bin/bash
# sparse-set A/B on one box: column (PIF_BOX=0) vs box (PIF_BOX=1) kernels
for cfg in "--N 256 --ppm 10" "--N 128 --ppm 64" "--N 128 --ppm 8" "--N 64 --ppm 64" "--N 64 --ppm 512"; do
  for b in 0 1; do
    PIF_BOX=$b python bench.py $cfg --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg box=$b', round(d['value']/1e9,3), 'Gps', round(d['ms_per_step'],2), 'ms', {k: round(v,2) for k,v in r['stage_ms'].items() if k in ('interp_push','spread','bin','fields')}, 'gather', round(r['frac'],3), 'spread', round(r['spread']['frac'],3))"
  done
done
