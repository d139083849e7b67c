#!/bin/bash
# long z-segments (cell table in shared memory, seg <= 127) vs the previous
# build (seg <= 31), with and without the weight cache, at several densities
L=paper_2605_10729_b200
for cfg in "--N 128 --ppm 64" "--N 256 --ppm 10" "--N 128 --ppm 128" "--N 64 --ppm 512"; do
  for lib in $L/lib_prev.so $L/libpifb200.so; do
    for wc in 0 1; do
      PIF_WEIGHT_CACHE=$wc PIF_B200_LIB=$lib python bench.py $cfg --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg', '$(basename $lib)', 'wc=$wc', round(d['value']/1e9,3), 'Gps', round(d['ms_per_step'],2), 'ms', {k: round(v,2) for k,v in r['stage_ms'].items() if k in ('interp_push','spread','bin')})"
    done
  done
done
