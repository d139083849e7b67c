"""Do the gather+push and the spread kernels fill each other's pipe gaps when
they run concurrently?  Two engines (2^26 particles each), engine A gathers
while engine B spreads, on two streams; compare with back-to-back."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_10729_b200 as pb  # noqa: E402
from paper_2605_10729_b200.engine import PifEngine  # noqa: E402

ppm = int(os.environ.get("PPM", "256"))
spec = pb.landau_spec(N=64, ppm=ppm, dt=0.003125)
M = spec.num_particles
plan = pb.make_plan(64, spec.L, 1e-7)
engs = []
for seed in (0, 1):
    e = PifEngine(plan, M, "cuda", q=spec.Q_e / M, m=-spec.Q_e / M, externals=spec.externals(),
                  dt=spec.dt)
    e.load_sampled(spec, (0, M), seed=seed)
    e.deposit(); e.solve_fields()
    for _ in range(2):
        e.step_once()
    engs.append(e)
A, B = engs
torch.cuda.synchronize()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def gather_a():
    with torch.cuda.stream(s1):
        A.interp_push(); A.rebin()


def spread_b():
    with torch.cuda.stream(s2):
        B.spread()


def seq():
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    gather_a()
    s2.wait_stream(s1)
    spread_b()


def conc():
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    gather_a()
    spread_b()


tg = timed(lambda: (s1.wait_stream(torch.cuda.current_stream()), gather_a()))
ts = timed(lambda: (s2.wait_stream(torch.cuda.current_stream()), spread_b()))
print(f"M={M}: gather+push {tg:.2f} ms, spread {ts:.2f} ms, back-to-back {timed(seq):.2f} ms, "
      f"concurrent {timed(conc):.2f} ms")
