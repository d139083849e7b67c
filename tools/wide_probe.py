"""Spread / gather timings for a few (N, M, eps) cases (PIF_FORCE_GENERIC /
PIF_FORCE_RING select the kernels):  python tools/wide_probe.py"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from tools.microbench import run_case, fp64_peak  # noqa: E402

peak = fp64_peak()
cases = [(64, 1 << 24, 1e-12), (128, 1 << 24, 1e-12), (32, 1 << 24, 1e-12), (64, 1 << 24, 1e-9),
         (64, 1 << 24, 1e-7), (64, 1 << 27, 1e-7)]
tag = " ".join(f"{k}={os.environ[k]}" for k in ("PIF_FORCE_GENERIC", "PIF_FORCE_RING") if k in os.environ)
for N, M, eps in cases:
    r = run_case(N, M, eps, "uniform", 3)
    sp = M * r["fs"] / r["ts"] / 1e12 / peak * 100
    gp = M * r["fg"] / r["tg"] / 1e12 / peak * 100
    print(f"{tag or 'default'} | {N}^3 2^{int(math.log2(M))} eps {eps:g} w={r['w']} | spread "
          f"{r['ts'] * 1e3:.2f} ms {sp:.1f}% | gather {r['tg'] * 1e3:.2f} ms {gp:.1f}%", flush=True)
