#!/bin/bash
# gather FMA sub-batches in pairs: A/B vs one at a time (p0), parity of the default build
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -q -x > gpurun_out/c50_tests.txt 2>&1
ab() {
  l=$1; lib=$2; shift 2
  if [ -n "$lib" ]; then export PIF_B200_LIB=$lib; else unset PIF_B200_LIB; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; st=r['stage_ms']
print('$l', '$*', round(d['value']/1e9,3), 'Gps', round(d['ms_per_step'],2), 'ms interp', round(st['interp_push'],2), 'spread', round(st['spread'],2), 'gfrac', round(r['frac'],3))" >> gpurun_out/c50_ab.txt 2>&1
  unset PIF_B200_LIB
}
for args in "--N 256 --ppm 10" "--N 128 --ppm 16" "--N 128 --ppm 64" "--N 64 --ppm 512"; do
  ab pairs "" $args
  ab p0 paper_2605_10729_b200/lib_p0.so $args
done
echo done
