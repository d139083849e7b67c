"""run_host timing breakdown: per-step time for several step counts / chunkings."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_10729_b200 as pb  # noqa: E402
from paper_2605_10729_b200.engine import PifEngine  # noqa: E402

spec = pb.landau_spec(N=64, ppm=int(os.environ.get("PPM", "512")), dt=0.003125)
M = spec.num_particles
plan = pb.make_plan(64, spec.L, 1e-7)
eng = PifEngine(plan, M, "cuda", q=spec.Q_e / M, m=-spec.Q_e / M, externals=spec.externals(),
                dt=spec.dt)
eng.load_sampled(spec, (0, M))
xd, vd = eng.to_id_order()
xh = torch.empty((M, 3), dtype=torch.float64, pin_memory=True)
vh = torch.empty((M, 3), dtype=torch.float64, pin_memory=True)
xh.copy_(xd)
vh.copy_(vd)
del xd, vd


def timed(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b)


eng.run_host(xh, vh, 0, 1)
for K, C in ((1, 16), (3, 16), (6, 16), (3, 1), (3, 64)):
    t = timed(lambda: eng.run_host(xh, vh, 0, K, n_chunks=C))
    print(f"K={K} chunks={C}: {t:.1f} ms total, {t / K:.1f} ms/step")


def steps_only():
    for _ in range(3):
        eng.step_once()


print(f"device steps: {timed(steps_only) / 3:.1f} ms/step")
xd, vd = eng.to_id_order()
print(f"to_id_order: {timed(lambda: eng.to_id_order(xd, vd)):.1f} ms")
ids = torch.arange(M, dtype=torch.int64, device='cuda')
print(f"load: {timed(lambda: eng.load(xd, vd, ids)):.1f} ms")
print(f"H2D x+v: {timed(lambda: (xd.copy_(xh, non_blocking=True), vd.copy_(vh, non_blocking=True))):.1f} ms")
print(f"D2H x+v: {timed(lambda: (xh.copy_(xd, non_blocking=True), vh.copy_(vd, non_blocking=True))):.1f} ms")
