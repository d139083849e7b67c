python bench.py --N 256 --ppm 10 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/paper256.json 2> gpurun_out/paper256.err
python -c "
import json; d=json.loads(open('gpurun_out/paper256.json').read().strip().splitlines()[-1]); print('256^3 ppm10', d['value'], d['ms_per_step'], d['roofline']['stage_ms'])"
python -m paper_2605_10729_b200.cli --benchmark landau --strategy pd --modes 64 --ppm 512 --steps 768 --ranks-space 1 --out-dir gpurun_out/cli_landau_64_2p27 --overwrite
