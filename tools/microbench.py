"""NUFFT type-1 / type-2 microbenchmark sweep (BASELINE.json configs[4]).

    python tools/microbench.py [--quick] > profiles/rNN_microbench.md

type-1 = points -> modes: binning (keys, scan, perm) + DMMA spreading + cuFFT D2Z
         + truncate/deconvolve (real strengths, the deposit path);
type-2 = modes -> points: padded symmetrised spectra + batched Z2D + DMMA gather
         of 3 real components (the gather_efield path, no push).
Uniform random points in [0, L)^3 (and a Penning-clustered variant), fp64, CUDA
events around each stage, median of reps.  Throughput in points/s and the FP64
roofline fraction of the spreading / gather kernels (2w^3+w^2 and 6w^3+w^2
flop per point against the live DFMA peak).
"""
import argparse
import ctypes
import math
import os
import statistics
import sys

# the NUFFT operator sweep times type 1 and type 2 as standalone transforms: no
# spread -> gather weight reuse (that belongs to the PD step, bench.py)
os.environ.setdefault("PIF_WEIGHT_CACHE", "0")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_10729_b200 as pb  # noqa: E402
from paper_2605_10729_b200 import _native  # noqa: E402
from paper_2605_10729_b200.engine import PifEngine  # noqa: E402


def timed(fn, reps):
    out = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        out.append(a.elapsed_time(b) * 1e-3)
    return statistics.median(out)


def fp64_peak():
    import bench
    return bench.fp64_peak_tflops(torch, torch.device("cuda", 0))


def run_case(N, M, eps, kind, reps):
    L = 2 * math.pi
    plan = pb.make_plan(N, L, eps)
    w = plan.window.w
    g = torch.Generator(device="cuda")
    g.manual_seed(N * 1000 + int(-math.log10(eps)))
    if kind == "uniform":
        x = torch.rand((M, 3), generator=g, dtype=torch.float64, device="cuda") * L
    else:   # Penning-like cloud: Gaussian (sigma L/12, L/25, L/8) about the centre
        sig = torch.tensor([L / 12, L / 25, L / 8], dtype=torch.float64, device="cuda")
        x = torch.remainder(L / 2 + torch.randn((M, 3), generator=g, dtype=torch.float64,
                                                device="cuda") * sig, L)
    v = torch.zeros_like(x)
    ids = torch.arange(M, dtype=torch.int64, device="cuda")
    eng = PifEngine(plan, M, "cuda", q=1.0 / M, m=1.0 / M, externals=pb.ExternalFieldsSpec(L=L),
                    dt=1.0)
    eng.load(x, v, ids)

    def type1():
        eng.load(x, v, ids)       # wrap + keys + scan + perm + work items
        eng.deposit()             # DMMA spread + D2Z + truncate/deconvolve

    def spread_only():
        eng.spread()

    E = torch.empty((M, 3), dtype=torch.float64, device="cuda")
    Ns = N ** 3
    rng = torch.Generator(device="cuda")
    rng.manual_seed(7)
    modes = [torch.complex(torch.randn((N, N, N), generator=rng, dtype=torch.float64,
                                       device="cuda"),
                           torch.zeros((N, N, N), dtype=torch.float64, device="cuda"))
             for _ in range(3)]

    def fields():
        _native.call("pif_fields_from_modes", eng.handle, modes[0].data_ptr(),
                     modes[1].data_ptr(), modes[2].data_ptr(), 0, eng.scalars.data_ptr(),
                     _native.stream_handle())

    def gather_only():
        cur = eng._soa()
        _native.call("pif_interp_perm", eng.handle, ctypes.byref(cur), eng.parts.perm.data_ptr(),
                     E.data_ptr(), _native.stream_handle())

    def type2():
        fields()
        gather_only()

    for f in (type1, type2):
        f()
    torch.cuda.synchronize()
    t1 = timed(type1, reps)
    ts = timed(spread_only, reps)
    t2 = timed(type2, reps)
    tg = timed(gather_only, reps)
    del eng, v, ids, E
    torch.cuda.empty_cache()
    # complex-strength type 1 / complex type 2 through the public API
    # (pb.type1 / pb.type2 on device tensors: binning + 2 spreads + C2C, or
    # C2C + gather, per call)
    cs = torch.complex(torch.randn(M, generator=rng, dtype=torch.float64, device="cuda"),
                       torch.randn(M, generator=rng, dtype=torch.float64, device="cuda"))
    fc = torch.complex(torch.randn((N, N, N), generator=rng, dtype=torch.float64, device="cuda"),
                       torch.randn((N, N, N), generator=rng, dtype=torch.float64, device="cuda"))
    pb.type1(plan, x, cs)
    pb.type2(plan, fc, x)
    t1c = timed(lambda: pb.type1(plan, x, cs), reps)
    t2c = timed(lambda: pb.type2(plan, fc, x), reps)
    del x, cs
    torch.cuda.empty_cache()
    return dict(N=N, M=M, eps=eps, w=w, kind=kind, t1=t1, ts=ts, t2=t2, tg=tg, t1c=t1c, t2c=t2c,
                fs=(2 * w ** 3 + w ** 2), fg=(6 * w ** 3 + w ** 2), modes=Ns)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    peak = fp64_peak()
    Ns = (32, 64, 128, 256)
    Ms = (1 << 20, 1 << 24, 1 << 27) if not a.quick else (1 << 20, 1 << 24)
    epss = (1e-6, 1e-12)
    print("# NUFFT microbenchmark sweep (BASELINE configs[4])\n")
    print(f"B200, fp64, FP64 peak measured live: {peak:.1f} TF/s. type-1 = bin + spread + "
          "D2Z + truncate; type-2 = padded Z2D (3 comps) + gather. Points/s = M / time.\n")
    print("| modes | points | eps (w) | layout | type-1 pts/s | spread | spread % FP64 | "
          "type-2 pts/s | gather | gather % FP64 | complex type-1 pts/s | complex type-2 pts/s |")
    print("|---|---|---|---|---:|---:|---:|---:|---:|---:|---:|---:|")
    for eps in epss:
        for N in Ns:
            for M in Ms:
                kinds = ("uniform", "clustered") if (N == 64 and M == 1 << 24) else ("uniform",)
                for kind in kinds:
                    if eps < 1e-8 and M > (1 << 24):
                        continue      # generic wide-window path: keep the sweep bounded
                    r = run_case(N, M, eps, kind, a.reps)
                    sp = M * r["fs"] / r["ts"] / 1e12 / peak * 100
                    gp = M * r["fg"] / r["tg"] / 1e12 / peak * 100
                    print(f"| {N}^3 | 2^{int(math.log2(M))} | {eps:g} ({r['w']}) | {kind} | "
                          f"{M / r['t1']:.3g} | {r['ts'] * 1e3:.2f} ms | {sp:.1f}% | "
                          f"{M / r['t2']:.3g} | {r['tg'] * 1e3:.2f} ms | {gp:.1f}% | "
                          f"{M / r['t1c']:.3g} | {M / r['t2c']:.3g} |", flush=True)


if __name__ == "__main__":
    main()
