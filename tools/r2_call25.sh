#!/bin/bash
# (1) full GPU suite (ring kernels up to w = 17), (2) ring split A/B,
# (3) Penning per-GPU-size sweep (gather efficiency vs particles per GPU),
# (4) warp-aggregated cell counts A/B.  ncu reports summarised on the box
# (gpurun_out must stay < 64 MiB).
mkdir -p gpurun_out
L=paper_2605_10729_b200
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/c25_tests.txt 2>&1
for ppm in 256 1024; do
  for lib in lib_base lib_redagg; do
    PIF_B200_LIB=$L/$lib.so timeout 600 python bench.py --kind penning --ppm $ppm --scaling strong \
      --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c25_pen_${ppm}_$lib.json \
      2> gpurun_out/c25_pen_${ppm}_$lib.err
  done
done
PIF_WEIGHT_CACHE=0 timeout 600 python bench.py --kind penning --ppm 1024 --scaling strong \
  --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c25_pen_1024_nocache.json 2>&1
for lib in lib_base lib_redagg; do
  PIF_B200_LIB=$L/$lib.so timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e \
    --no-cpu-baseline > gpurun_out/c25_landau_$lib.json 2> gpurun_out/c25_landau_$lib.err
done
for c in "32 24 1e-12" "64 24 1e-12" "32 24 1e-13" "64 24 1e-13" "32 24 1e-14" "64 24 1e-15" \
         "32 24 1e-16" "64 24 1e-16" "128 24 1e-15"; do
  for lib in $L/lib_prev.so $L/libpifb200.so $L/lib_split12.so; do
    echo -n "$(basename $lib) "; PIF_B200_LIB=$lib timeout 300 python tools/mb_case.py $c 2>&1 | tail -1
  done
done > gpurun_out/c25_ring_ab.txt
for t in pen1024 pen256; do
  ppm=${t#pen}
  PIF_B200_LIB=$L/lib_base.so bash tools/profile_hot.sh $t --kind penning --ppm $ppm --scaling strong
  python tools/ncu_summary.py full gpurun_out/prof_$t.ncu-rep > gpurun_out/c25_full_$t.md 2>&1
  python tools/ncu_summary.py launches gpurun_out/launches_$t.csv > gpurun_out/c25_launches_$t.md 2>&1
  ncu -i gpurun_out/prof_$t.ncu-rep --page source --csv --print-source sass -k regex:interp_mma \
    > gpurun_out/src_$t.csv 2>/dev/null
  python tools/ncu_sass_stalls.py gpurun_out/src_$t.csv > gpurun_out/c25_stalls_$t.txt 2>&1
  rm -f gpurun_out/src_$t.csv
  rm -f gpurun_out/prof_$t.ncu-rep
done
du -sh gpurun_out
echo done
