#!/bin/bash
# re-entry check of HEAD: GPU suite + bench line
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/c33_tests.txt 2>&1
timeout 900 python bench.py > gpurun_out/c33_bench.json 2> gpurun_out/c33_bench.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c33_smoke.txt 2>&1
echo done
