#!/bin/bash
# final validation after the unroll change: GPU suite, smoke, bench line, sparse line
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c61_tests.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c61_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/c61_bench.json 2> gpurun_out/c61_bench.err
timeout 600 python bench.py --N 256 --ppm 10 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c61_sparse.json 2> gpurun_out/c61_sparse.err
echo done
