#!/bin/bash
# unrolled cursor binning: A/B of the bin stage + parity
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py tests/test_gpu_determinism.py -q -x > gpurun_out/c55_tests.txt 2>&1
ab() {
  l=$1; lib=$2; shift 2
  if [ -n "$lib" ]; then export PIF_B200_LIB=$lib; else unset PIF_B200_LIB; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; st=r['stage_ms']
print('$l', '$*', round(d['value']/1e9,3), 'Gps', round(d['ms_per_step'],3), 'ms bin', round(st['bin'],3), 'interp', round(st['interp_push'],2), 'spread', round(st['spread'],2))" >> gpurun_out/c55_ab.txt 2>&1
  unset PIF_B200_LIB
}
for rep in 1 2; do
for args in "--N 64 --ppm 512" "--N 256 --ppm 10"; do
  ab new "" $args
  ab old paper_2605_10729_b200/lib_prevbin.so $args
done
done
echo done
