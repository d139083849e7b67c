"""Which part of bench.py's preamble changes run_host's copy overlap?
Variants by env: PRE_PROBE=1 (DFMA probe), PRE_STEPS=n (device steps),
PRE_SMI=1 (nvidia-smi sampler running during the device steps)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_10729_b200 as pb  # noqa: E402
from paper_2605_10729_b200.engine import PifEngine  # noqa: E402

spec = pb.landau_spec(N=64, ppm=512, dt=0.003125)
M = spec.num_particles
plan = pb.make_plan(64, spec.L, 1e-7)
eng = PifEngine(plan, M, "cuda", q=spec.Q_e / M, m=-spec.Q_e / M, externals=spec.externals(),
                dt=spec.dt)
eng.load_sampled(spec, (0, M))
if os.environ.get("PRE_PROBE") == "1":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    print("probe", bench.fp64_peak_tflops(torch, torch.device("cuda", 0)))
smi = None
if os.environ.get("PRE_SMI") == "1":
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv", "-lms", "100"],
                           stdout=subprocess.DEVNULL)
n = int(os.environ.get("PRE_STEPS", "0"))
if n:
    eng.particle_diag(); eng.deposit(); eng.allreduce(); eng.solve_fields()
    for _ in range(n):
        eng.step_once()
    torch.cuda.synchronize()
if smi is not None:
    smi.terminate()
    smi.wait()
xd0, vd0 = eng.to_id_order()
xh = torch.empty((M, 3), dtype=torch.float64, pin_memory=True)
vh = torch.empty((M, 3), dtype=torch.float64, pin_memory=True)
xh.copy_(xd0)
vh.copy_(vd0)
del xd0, vd0
eng.run_host(xh, vh, 0, 1)
torch.cuda.synchronize()
tr = []
eng.run_host(xh, vh, 0, 4, trace=tr)
torch.cuda.synchronize()
for s, evs in enumerate(tr):
    print("step", s, " ".join(f"{evs[0].elapsed_time(x):.1f}" for x in evs[:7]))
