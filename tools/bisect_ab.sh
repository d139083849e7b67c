#!/bin/bash
# bisect the sparse / dense gather regression across round-2 commits
L=paper_2605_10729_b200
for cfg in "--N 256 --ppm 10" "--N 64 --ppm 512"; do
  for tag in ev bank halo tma1 head; do
    lib=$L/lib_$tag.so; [ $tag = head ] && lib=$L/libpifb200.so
    PIF_B200_LIB=$lib python bench.py $cfg --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg', '$tag', round(d['value']/1e9,3), 'Gps', round(d['ms_per_step'],2), 'ms', {k: round(v,2) for k,v in r['stage_ms'].items() if k in ('interp_push','spread','bin','fields')})"
  done
done
