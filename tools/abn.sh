#!/bin/bash
# tools/abn.sh reps lib1.so lib2.so ...  — alternate bench runs over several libraries on one box
reps=$1; shift
for i in $(seq $reps); do
  for v in "$@"; do
    PIF_B200_LIB=$v python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $v)', round(d['value']/1e9,3), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['roofline']['stage_ms'].items() if k in ('interp_push','spread','bin')})"
  done
done
