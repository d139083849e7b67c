#!/bin/bash
# Strong scaling of a fixed global workload over 1..G GPUs (powers of two).
#   bash tools/strong_scaling.sh G N PPM TAG   (writes gpurun_out/TAG_nN.json)
G=${1:-4}; NM=${2:-64}; PPM=${3:-4096}; TAG=${4:-strong}
mkdir -p gpurun_out
n=1
while [ $n -le $G ]; do
  if [ $n -eq 1 ]; then
    python bench.py --N $NM --ppm $PPM --scaling strong --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_n1.json 2> gpurun_out/${TAG}_n1.err
  else
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700 + n)) \
      bench.py --gpus $n --N $NM --ppm $PPM --scaling strong --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_n$n.json 2> gpurun_out/${TAG}_n$n.err
  fi
  python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_n$n.json').read().strip().splitlines()[-1]); print('N=$n', round(d['value']/1e9,3), 'G particle-steps/s', round(d['ms_per_step'],2), 'ms/step', {k: round(v,2) for k,v in d['roofline']['stage_ms'].items()})"
  n=$((n * 2))
done
