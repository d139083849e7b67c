"""Phase split of the warp-specialised gather (-DPIF_PHASE_TIMING build)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_10729_b200 as pb  # noqa: E402
from paper_2605_10729_b200 import _native  # noqa: E402
from paper_2605_10729_b200.engine import PifEngine  # noqa: E402
from paper_2605_10729_b200.samplers import sample_device  # noqa: E402

spec = pb.landau_spec(N=64, ppm=512, dt=0.003125)
M = spec.num_particles
plan = pb.make_plan(64, spec.L, 1e-7)
x, v, ids = sample_device(spec, (0, M), "cuda")
eng = PifEngine(plan, M, "cuda", q=spec.Q_e / M, m=-spec.Q_e / M, externals=spec.externals(),
                dt=spec.dt)
eng.load(x, v, ids)
del x, v, ids
eng.deposit(); eng.solve_fields()
for _ in range(2):
    eng.step_once()
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 8)()
_native.call("pif_debug_phase_cycles", buf)
eng.interp_push()
torch.cuda.synchronize()
_native.call("pif_debug_phase_cycles", buf)
c = max(buf[5], 1)
print(f"chunks {buf[5]}; per chunk: particle warp weights {buf[0]/c:.0f} push {buf[1]/c:.0f} "
      f"wait-E {buf[2]/c:.0f} | MMA warp gather {buf[6]/c:.0f} wait-ready {buf[7]/c:.0f}")
