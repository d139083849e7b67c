#!/bin/bash
# tools/envsweep.sh "BENCH ARGS" VAR v1 v2 ...  — bench once per value of env VAR (one box)
args=$1; var=$2; shift 2
for v in "$@"; do
  env $var=$v python bench.py $args --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$var=$v', round(d['value']/1e9,3), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['roofline']['stage_ms'].items() if k in ('interp_push','spread','bin')})"
done
