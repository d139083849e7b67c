"""Event timeline of PifEngine.run_host-style stepping (where the e2e time goes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_10729_b200 as pb  # noqa: E402
from paper_2605_10729_b200 import _native  # noqa: E402
from paper_2605_10729_b200.engine import PifEngine  # noqa: E402

spec = pb.landau_spec(N=64, ppm=512, dt=0.003125)
M = spec.num_particles
plan = pb.make_plan(64, spec.L, 1e-7)
eng = PifEngine(plan, M, "cuda", q=spec.Q_e / M, m=-spec.Q_e / M, externals=spec.externals(),
                dt=spec.dt)
eng.load_sampled(spec, (0, M))
xd0, vd0 = eng.to_id_order()
xh = torch.empty((M, 3), dtype=torch.float64, pin_memory=True)
vh = torch.empty((M, 3), dtype=torch.float64, pin_memory=True)
xh.copy_(xd0)
vh.copy_(vd0)
del xd0, vd0
xd = torch.empty((M, 3), dtype=torch.float64, device="cuda")
vd = torch.empty((M, 3), dtype=torch.float64, device="cuda")
main = torch.cuda.current_stream()
down, up = torch.cuda.Stream(), torch.cuda.Stream()
C = int(os.environ.get("CHUNKS", "16"))
step = -(-M // C)
bounds = [(i, min(M, i + step)) for i in range(0, M, step)]
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
marks = []
phases = []
t0 = ev()
t0.record()
up.wait_stream(main)
with torch.cuda.stream(up):
    xd.copy_(xh, non_blocking=True)
    vd.copy_(vh, non_blocking=True)
K = 4
for s in range(K):
    main.wait_stream(up)
    a = ev(); a.record(main)
    eng.load_aos(xd, vd, 0)
    a1 = ev(); a1.record(main)
    eng.deposit(); eng.allreduce(); eng.solve_fields()
    a2 = ev(); a2.record(main)
    if os.environ.get("NOMIRROR") != "1":
        _native.call("pif_set_id_order_output", eng.handle, xd.data_ptr(), vd.data_ptr(), 0)
    eng.gather_push()
    _native.call("pif_set_id_order_output", eng.handle, None, None, 0)
    b = ev(); b.record(main)
    phases.append((a, a1, a2, b))
    down.wait_stream(main)
    last = s == K - 1
    for i0, i1 in bounds:
        with torch.cuda.stream(down):
            xh[i0:i1].copy_(xd[i0:i1], non_blocking=True)
            vh[i0:i1].copy_(vd[i0:i1], non_blocking=True)
        if not last:
            up.wait_stream(down)
            with torch.cuda.stream(up):
                xd[i0:i1].copy_(xh[i0:i1], non_blocking=True)
                vd[i0:i1].copy_(vh[i0:i1], non_blocking=True)
    c = ev(); c.record(down)
    d = ev(); d.record(up)
    marks.append((a, b, c, d))
torch.cuda.synchronize()
for s, (a, a1, a2, b) in enumerate(phases):
    print(f"step {s}: load_aos+bin {a.elapsed_time(a1):.1f} ms, deposit+solve {a1.elapsed_time(a2):.1f} ms, "
          f"gather+push(+mirror) {a2.elapsed_time(b):.1f} ms")
for s, (a, b, c, d) in enumerate(marks):
    print(f"step {s}: compute start {t0.elapsed_time(a):8.1f}  compute end {t0.elapsed_time(b):8.1f}"
          f"  D2H end {t0.elapsed_time(c):8.1f}  H2D end {t0.elapsed_time(d):8.1f} ms")
