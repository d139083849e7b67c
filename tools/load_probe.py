import os, sys
sys.path.insert(0, "/root/repo")
import torch, ctypes
import paper_2605_10729_b200 as pb
from paper_2605_10729_b200 import _native
from paper_2605_10729_b200.engine import PifEngine
spec = pb.landau_spec(N=64, ppm=512, dt=0.003125)
M = spec.num_particles
plan = pb.make_plan(64, spec.L, 1e-7)
eng = PifEngine(plan, M, "cuda", q=spec.Q_e / M, m=-spec.Q_e / M, externals=spec.externals(), dt=spec.dt)
eng.load_sampled(spec, (0, M))
xd, vd = eng.to_id_order()
def t(fn, reps=3):
    best=1e9
    for _ in range(reps):
        torch.cuda.synchronize(); a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); best=min(best,a.elapsed_time(b))
    return best
def load_only():
    cur = eng._soa()
    _native.call("pif_load_aos", eng.handle, xd.data_ptr(), vd.data_ptr(), 0, ctypes.byref(cur), eng.parts.key.data_ptr(), eng.parts.rank.data_ptr(), eng._stream())
def bin_only():
    eng._bin()
print("load_aos", t(lambda: (load_only(), bin_only())), "ms (load+bin)")
print("bin only after load", t(bin_only))
print("load only (counts accumulate)", t(load_only))
