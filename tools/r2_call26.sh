#!/bin/bash
# push cell counts: per-lane RED (lib_base) vs __match_any aggregation (lib_redagg)
# vs runs of equal keys (lib_runs = HEAD); Landau default + Penning 2^28, two rounds.
mkdir -p gpurun_out
L=paper_2605_10729_b200
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_scale_parity.py -m gpu -q -x > gpurun_out/c26_tests.txt 2>&1
for rep in 1 2; do
  for lib in lib_base lib_runs lib_redagg; do
    PIF_B200_LIB=$L/$lib.so timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e \
      --no-cpu-baseline > gpurun_out/c26_landau_${lib}_$rep.json 2> /dev/null
  done
done
for lib in lib_base lib_runs; do
  PIF_B200_LIB=$L/$lib.so timeout 600 python bench.py --kind penning --ppm 1024 --scaling strong \
    --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c26_pen_1024_$lib.json 2> /dev/null
done
for c in "32 24 1e-11" "64 24 1e-11" "64 24 1e-12"; do
  for lib in $L/lib_prev.so $L/libpifb200.so; do
    echo -n "$(basename $lib) "; PIF_B200_LIB=$lib timeout 300 python tools/mb_case.py $c 2>&1 | tail -1
  done
done > gpurun_out/c26_ring.txt
echo done
