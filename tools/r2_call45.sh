#!/bin/bash
# 4-GPU box: weak scaling lines (default bench config per GPU) with the split e2e
mkdir -p gpurun_out
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n bench.py --gpus $n --steps 20 --warmup 3 > gpurun_out/c45_weak_n$n.json 2> gpurun_out/c45_weak_n$n.err
done
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/c45_weak_n1.json 2> gpurun_out/c45_weak_n1.err
echo done
