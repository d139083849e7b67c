#!/bin/bash
# round-2 multi-GPU evidence on one G-GPU box (G = 4): NCCL thread-rank tests,
# north-star strong scaling (64^3 / 2^30), configs[3] strong scaling
# (128^3 / 2^30), weak scaling (2^27 per GPU), and the weight-cache A/B.
G=${1:-4}
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/r2m_smi.txt
python -m pytest tests/test_gpu_multi.py tests/test_gpu_determinism.py -v > gpurun_out/r2m_tests.txt 2>&1
bash tools/north_star_scaling.sh $G > gpurun_out/r2m_ns.txt 2>&1
bash tools/strong_scaling.sh $G 128 512 cfg4 > gpurun_out/r2m_cfg4.txt 2>&1
for n in 2 4; do
  [ $n -le $G ] || continue
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29800 + n)) bench.py --gpus $n --no-cpu-baseline > gpurun_out/r2m_weak_n$n.json \
    2> gpurun_out/r2m_weak_n$n.err
done
# configs[2]: Penning 64^3, 2^28 particles (strong over 1/2/4 of the 8 GPUs it names)
for n in 1 2 4; do
  [ $n -le $G ] || continue
  if [ $n -eq 1 ]; then
    python bench.py --kind penning --ppm 1024 --scaling strong --steps 5 --warmup 3 --no-e2e \
      --no-cpu-baseline > gpurun_out/r2m_penning_n1.json 2> gpurun_out/r2m_penning_n1.err
  else
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29900 + n)) bench.py --gpus $n --kind penning --ppm 1024 --scaling strong \
      --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2m_penning_n$n.json \
      2> gpurun_out/r2m_penning_n$n.err
  fi
done
