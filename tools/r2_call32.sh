#!/bin/bash
# HEAD: GPU suite, bench line, e2e timeline (agg check through mapped memory), microbench sweep
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/c32_tests.txt 2>&1
timeout 900 python bench.py > gpurun_out/c32_bench.json 2> gpurun_out/c32_bench.err
timeout 600 python tools/e2e_timeline.py 27 16 > gpurun_out/c32_tl.txt 2>&1
timeout 2400 python tools/microbench.py > gpurun_out/c32_microbench.md 2> gpurun_out/c32_microbench.err
echo done
