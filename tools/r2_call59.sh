#!/bin/bash
# final check after the heavy-cell rule: full GPU suite, microbench, bench line, sparse line
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c59_tests.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c59_smoke.txt 2>&1
timeout 2400 python tools/microbench.py > gpurun_out/c59_microbench.md 2> gpurun_out/c59_microbench.err
timeout 900 python bench.py > gpurun_out/c59_bench.json 2> gpurun_out/c59_bench.err
timeout 600 python bench.py --N 256 --ppm 10 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c59_sparse.json 2> gpurun_out/c59_sparse.err
echo done
