#!/bin/bash
# merged-column spread: parity tests, then A/B by density (spread stage ms, whole step)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_scale_parity.py -q -x > gpurun_out/c46_tests.txt 2>&1
ab() {  # label env args
  l=$1; e=$2; shift 2
  env $e timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; st=r['stage_ms']
print('$l', '$*', round(d['value']/1e9,3), 'Gps', round(d['ms_per_step'],2), 'ms spread', round(st['spread'],2), 'bin', round(st['bin'],2), 'interp', round(st['interp_push'],2), 'sfrac', round(r['spread']['frac'],3))" >> gpurun_out/c46_ab.txt 2>&1
}
for args in "--N 256 --ppm 10" "--N 128 --ppm 64" "--N 128 --ppm 128" "--N 64 --ppm 64" "--N 64 --ppm 512"; do
  for m in 0 2 4; do ab "merge=$m" "PIF_SPREAD_MERGE=$m" $args; done
done
echo done
