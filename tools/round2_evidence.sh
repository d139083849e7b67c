#!/bin/bash
# Round-2 evidence on one GPU (outputs gpurun_out/ev_*): GPU test suite, the
# default bench line, ncu launch list + full capture of the hot kernels, the
# NUFFT microbenchmark sweep (configs[4]), Penning, the paper's sparse run and
# its gather DRAM bytes.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/ev_gpu.txt 2>&1
python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err
python bench.py --kind penning --no-cpu-baseline > gpurun_out/ev_penning.json 2>/dev/null
python bench.py --N 256 --ppm 10 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ev_sparse.json 2>/dev/null
bash tools/profile_hot.sh final
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"interp_mma|spread_mma" -s 2 -c 2 --csv python bench.py --N 256 --ppm 10 --steps 1 \
    --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ev_sparse_ncu.csv 2> gpurun_out/ev_sparse_ncu.err
python tools/microbench.py > gpurun_out/ev_microbench.md 2> gpurun_out/ev_microbench.err
