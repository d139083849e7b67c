#!/bin/bash
# split host-streamed step: parity tests, timeline, bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "run_host or split" > gpurun_out/c35_tests.txt 2>&1
timeout 600 python tools/e2e_timeline.py 27 16 > gpurun_out/c35_tl16.txt 2>&1
timeout 900 python bench.py > gpurun_out/c35_bench.json 2> gpurun_out/c35_bench.err
echo done
