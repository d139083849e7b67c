"""One microbenchmark case (tools/microbench.py run_case) for A/B runs:
    python tools/mb_case.py N log2M eps [kind]"""
import math
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
from microbench import fp64_peak, run_case  # noqa: E402

N, lm, eps = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
kind = sys.argv[4] if len(sys.argv) > 4 else "uniform"
peak = fp64_peak()
r = run_case(N, 1 << lm, eps, kind, 3)
M = 1 << lm
print(f"N={N} M=2^{lm} eps={eps:g} w={r['w']}: spread {r['ts'] * 1e3:.2f} ms "
      f"({M * r['fs'] / r['ts'] / 1e12 / peak * 100:.1f}%), gather {r['tg'] * 1e3:.2f} ms "
      f"({M * r['fg'] / r['tg'] / 1e12 / peak * 100:.1f}%), type1 {r['t1'] * 1e3:.2f} ms")
