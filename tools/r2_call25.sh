#!/bin/bash
# (1) full GPU suite (ring kernels up to w = 17), (2) ring split A/B,
# (3) Penning per-GPU-size sweep (gather efficiency vs particles per GPU).
mkdir -p gpurun_out
L=paper_2605_10729_b200
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/c25_tests.txt 2>&1
for c in "32 24 1e-12" "64 24 1e-12" "32 24 1e-13" "64 24 1e-13" "32 24 1e-14" "64 24 1e-15" \
         "32 24 1e-16" "64 24 1e-16" "128 24 1e-15"; do
  for lib in $L/lib_prev.so $L/libpifb200.so $L/lib_split12.so; do
    echo -n "$(basename $lib) "; PIF_B200_LIB=$lib timeout 300 python tools/mb_case.py $c 2>&1 | tail -1
  done
done > gpurun_out/c25_ring_ab.txt
for ppm in 256 512 1024; do
  for wc in auto 0; do
    PIF_WEIGHT_CACHE=$wc timeout 600 python bench.py --kind penning --ppm $ppm --scaling strong \
      --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c25_pen_${ppm}_$wc.json \
      2> gpurun_out/c25_pen_${ppm}_$wc.err
  done
done
bash tools/profile_hot.sh pen1024 --kind penning --ppm 1024 --scaling strong
bash tools/profile_hot.sh pen256 --kind penning --ppm 256 --scaling strong
echo done
