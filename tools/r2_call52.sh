#!/bin/bash
# 2 GPUs after the merged spread: NCCL process / thread-rank tests
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -rs > gpurun_out/c52_multi.txt 2>&1
echo done
