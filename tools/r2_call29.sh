#!/bin/bash
# HEAD (automatic push-count aggregation, ring thresholds, split from w = 13):
# full GPU suite, A/B vs lib_base (per-lane counts always), microbench sweep.
mkdir -p gpurun_out
L=paper_2605_10729_b200
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/c29_tests.txt 2>&1
for rep in 1 2; do
  for lib in lib_base lib_agg; do
    PIF_B200_LIB=$L/$lib.so timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e \
      --no-cpu-baseline > gpurun_out/c29_landau_${lib}_$rep.json 2> /dev/null
  done
done
for lib in lib_base lib_agg; do
  for ppm in 1024 512; do
    PIF_B200_LIB=$L/$lib.so timeout 600 python bench.py --kind penning --ppm $ppm --scaling strong \
      --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c29_pen_${ppm}_$lib.json 2> /dev/null
  done
  PIF_B200_LIB=$L/$lib.so timeout 600 python bench.py --N 64 --ppm 4096 --scaling strong --steps 3 \
    --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c29_l2p30_$lib.json 2> /dev/null
done
timeout 1800 python tools/microbench.py > gpurun_out/c29_microbench.md 2> gpurun_out/c29_microbench.err
echo done
timeout 600 python tools/e2e_timeline.py 27 16 > gpurun_out/c29_e2e_timeline.txt 2>&1
timeout 300 python tools/pcie_probe.py > gpurun_out/c29_pcie.txt 2>&1
echo done2
for rep in 1 2; do
  for lib in lib_chains6 lib_chains3; do
    PIF_B200_LIB=$L/$lib.so timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e \
      --no-cpu-baseline > gpurun_out/c29_landau_${lib}_$rep.json 2> /dev/null
  done
done
echo done3
