"""Where the e2e time goes: event timeline of PifEngine.run_host at the bench
workload (Landau 64^3, 2^27 particles unless argv[1] gives log2 M).

  python tools/e2e_timeline.py [log2M] [n_chunks]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_10729_b200 as pb  # noqa: E402
from paper_2605_10729_b200.engine import PifEngine  # noqa: E402

lm = int(sys.argv[1]) if len(sys.argv) > 1 else 27
chunks = int(sys.argv[2]) if len(sys.argv) > 2 else 16
ppm = (1 << lm) // 64 ** 3
spec = pb.landau_spec(N=64, ppm=ppm, dt=0.003125)
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
wh = torch.empty(4, dtype=torch.float64, pin_memory=True)   # as bench.py: W per step
eng.run_host(xh, vh, 0, 1, energy_out=wh, n_chunks=chunks)
torch.cuda.synchronize()
tr = []
t0 = torch.cuda.Event(enable_timing=True)
t0.record()
eng.run_host(xh, vh, 0, 4, energy_out=wh, n_chunks=chunks, trace=tr)
torch.cuda.synchronize()
print(f"M = 2^{lm}, {chunks} chunks; ms from the first step's start")
names = ("start", "x in", "fields", "v in", "push", "D2H end", "H2D end")
print("step " + "".join(f"{n:>10}" for n in names))
for s, evs in enumerate(tr):
    print(f"{s:4d} " + "".join(f"{t0.elapsed_time(e):10.1f}" for e in evs[:7]))
for s, evs in enumerate(tr):
    st, xi, fi, vi, pu, dn, upd, tb, tp, td = evs
    print(f"step {s}: load_aos+bin {xi.elapsed_time(tb):.1f}, permute {tb.elapsed_time(tp):.1f},"
          f" deposit {tp.elapsed_time(td):.1f}, allreduce+solve {td.elapsed_time(fi):.1f}")
for s, evs in enumerate(tr):
    st, xi, fi, vi, pu, dn, upd = evs[:7]
    print(f"step {s}: wait x {st.elapsed_time(xi):.1f}, load+bin+deposit+solve {xi.elapsed_time(fi):.1f},"
          f" wait v {fi.elapsed_time(vi):.1f}, v load+gather+push {vi.elapsed_time(pu):.1f},"
          f" push->D2H end {pu.elapsed_time(dn):.1f}, push->H2D end {pu.elapsed_time(upd):.1f}")
