#!/bin/bash
# e2e with NUMA-local pinned staging vs without, 1 and 4 ranks
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/c53_topo.txt 2>&1
lscpu > gpurun_out/c53_lscpu.txt 2>&1
for numa in 1 0; do
  PIF_E2E_NUMA=$numa timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2956$numa bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c53_n4_numa$numa.json 2> gpurun_out/c53_n4_numa$numa.err
  PIF_E2E_NUMA=$numa timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c53_n1_numa$numa.json 2> gpurun_out/c53_n1_numa$numa.err
done
echo done
