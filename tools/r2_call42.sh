#!/bin/bash
# 2 GPUs: NCCL tests + torchrun bench (weak, with the split e2e)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/c42_multi.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/c42_bench_n2.json 2> gpurun_out/c42_bench_n2.err
echo done
