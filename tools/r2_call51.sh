#!/bin/bash
# final validation: GPU suite, smoke, default + sparse bench lines, ncu of the sparse kernels
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c51_tests.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c51_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/c51_bench.json 2> gpurun_out/c51_bench.err
timeout 600 python bench.py --N 256 --ppm 10 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c51_sparse.json 2> gpurun_out/c51_sparse.err
ncu --set full --import-source on --clock-control none -k regex:"spread_merged|interp_mma" -s 2 -c 2 \
    -f -o gpurun_out/prof_c51_sparse python bench.py --N 256 --ppm 10 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c51.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex_op_red.sum --clock-control none -k regex:"spread_merged|spread_mma|interp_mma" -s 4 -c 6 --csv \
    --log-file gpurun_out/c51_sparse_dram.csv python bench.py --N 256 --ppm 10 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c51b.log 2>&1
echo done
