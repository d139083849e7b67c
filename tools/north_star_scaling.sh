#!/bin/bash
# North-star strong scaling: Landau 64^3 modes, 2^30 particles total, N = 1..G GPUs.
#   bash tools/north_star_scaling.sh G [extra bench args]   (writes gpurun_out/ns_nN.json)
G=${1:-4}; shift
mkdir -p gpurun_out
n=1
while [ $n -le $G ]; do
  if [ $n -eq 1 ]; then
    python bench.py --N 64 --ppm 4096 --scaling strong --steps 3 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/ns_n1.json 2> gpurun_out/ns_n1.err
  else
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + n)) \
      bench.py --gpus $n --N 64 --ppm 4096 --scaling strong --steps 3 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/ns_n$n.json 2> gpurun_out/ns_n$n.err
  fi
  python -c "
import json; d=json.loads(open('gpurun_out/ns_n$n.json').read().strip().splitlines()[-1]); print('N=$n', round(d['value']/1e9,3), 'G particle-steps/s', round(d['ms_per_step'],2), 'ms/step', {k: round(v,2) for k,v in d['roofline']['stage_ms'].items()})"
  n=$((n * 2))
done
