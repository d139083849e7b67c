#!/bin/bash
# tools/ab2.sh "BENCH ARGS" lib1.so lib2.so ...  — one bench per library with the given args
args=$1; shift
for v in "$@"; do
  PIF_B200_LIB=$v python bench.py $args --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $v)', '${args}'[:18], round(d['value']/1e9,3), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['roofline']['stage_ms'].items() if k in ('interp_push','spread','bin')})"
done
