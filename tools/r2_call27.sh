#!/bin/bash
# dense-segment-only run aggregation of the push's cell counts (lib_runs2 = HEAD)
# vs per-lane REDs (lib_base): Landau 2^27 (64/cell), Landau 2^30 (512/cell),
# Penning 2^28, Penning 2^26; plus the parity/determinism tests on HEAD.
mkdir -p gpurun_out
L=paper_2605_10729_b200
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_scale_parity.py tests/test_gpu_plugin.py -m gpu -q -x > gpurun_out/c27_tests.txt 2>&1
for rep in 1 2; do
  for lib in lib_base lib_runs2; do
    PIF_B200_LIB=$L/$lib.so timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e \
      --no-cpu-baseline > gpurun_out/c27_landau_${lib}_$rep.json 2> /dev/null
  done
done
for lib in lib_base lib_runs2; do
  PIF_B200_LIB=$L/$lib.so timeout 600 python bench.py --N 64 --ppm 4096 --scaling strong --steps 3 \
    --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c27_l2p30_$lib.json 2> /dev/null
  for ppm in 1024 256; do
    PIF_B200_LIB=$L/$lib.so timeout 600 python bench.py --kind penning --ppm $ppm --scaling strong \
      --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c27_pen_${ppm}_$lib.json 2> /dev/null
  done
done
echo done
