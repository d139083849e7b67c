#!/bin/bash
# final-candidate check: GPU suite, smoke, default bench line
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/c44_tests.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c44_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/c44_bench.json 2> gpurun_out/c44_bench.err
echo done
