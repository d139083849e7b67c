#!/bin/bash
# final code on 2 GPUs: NCCL tests + torchrun bench line (the driver's scaling path)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -rs > gpurun_out/c62_multi.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 2 > gpurun_out/c62_bench_n2.json 2> gpurun_out/c62_bench_n2.err
echo done
