#!/bin/bash
# merged perm by per-cell copy: parity, microbench sweep, sparse bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x > gpurun_out/c57_tests.txt 2>&1
timeout 2400 python tools/microbench.py > gpurun_out/c57_microbench.md 2> gpurun_out/c57_microbench.err
timeout 600 python bench.py --N 256 --ppm 10 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c57_sparse.json 2> gpurun_out/c57_sparse.err
for m in 0 -1; do
  for args in "--N 128 --ppm 64" "--N 128 --ppm 24"; do
    PIF_WEIGHT_CACHE=0 PIF_SPREAD_MERGE=$m timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline $args 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); st=d['roofline']['stage_ms']
print('cache=0 merge=$m', '$args', round(d['value']/1e9,3), 'Gps spread', round(st['spread'],2), 'interp', round(st['interp_push'],2))" >> gpurun_out/c57_ab.txt 2>&1
  done
done
echo done
