"""Per-phase cycle split of the gather+push kernel (needs a -DPIF_PHASE_TIMING build):
    PIF_B200_LIB=paper_2605_10729_b200/libpif_phase.so python tools/phase_timing.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_10729_b200 as pb  # noqa: E402
from paper_2605_10729_b200 import _native  # noqa: E402
from paper_2605_10729_b200.engine import PifEngine  # noqa: E402
from paper_2605_10729_b200.samplers import sample_device  # noqa: E402

spec = pb.landau_spec(N=64, ppm=int(os.environ.get("PPM", "512")), dt=0.003125)
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
w, g, p, chunks, parts = buf[0], buf[1], buf[2], buf[3], buf[4]
tot = w + g + p
print(f"chunks {chunks} particles {parts}; warp-cycles per chunk: weights {w/chunks:.0f} "
      f"gather {g/chunks:.0f} push {p/chunks:.0f}; shares {100*w/tot:.1f}/{100*g/tot:.1f}/{100*p/tot:.1f}%")
