#!/bin/bash
# end-of-round validation of HEAD: GPU suite, smoke, default bench line, sparse line, launch list
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c54_tests.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c54_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/c54_bench.json 2> gpurun_out/c54_bench.err
timeout 600 python bench.py --N 256 --ppm 10 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c54_sparse.json 2> gpurun_out/c54_sparse.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c54_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c54_ncu_l.log 2>&1
echo done
