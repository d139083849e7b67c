#!/bin/bash
# final: GPU suite, smoke, default bench line, cache-off merge threshold A/B, microbench sweep
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c56_tests.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c56_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/c56_bench.json 2> gpurun_out/c56_bench.err
for m in 0 -1; do
  for args in "--N 128 --ppm 64" "--N 128 --ppm 32" "--N 128 --ppm 24"; do
    PIF_WEIGHT_CACHE=0 PIF_SPREAD_MERGE=$m timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline $args 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); st=d['roofline']['stage_ms']
print('cache=0 merge=$m', '$args', round(d['value']/1e9,3), 'Gps spread', round(st['spread'],2), 'interp', round(st['interp_push'],2))" >> gpurun_out/c56_ab.txt 2>&1
  done
done
timeout 2400 python tools/microbench.py > gpurun_out/c56_microbench.md 2> gpurun_out/c56_microbench.err
echo done
