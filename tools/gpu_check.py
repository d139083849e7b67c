"""Stage-by-stage GPU vs oracle check (diagnostic script; prints errors).

    python tools/gpu_check.py
"""
import os
import sys
import time
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_10729_b200 as pb  # noqa: E402
from oracle import pif_oracle as o  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def stage(name, fn):
    t = time.time()
    try:
        r = fn()
        print(f"[ok ] {name}: {r}  ({time.time() - t:.2f}s)", flush=True)
    except Exception:
        print(f"[ERR] {name}", flush=True)
        traceback.print_exc()


def main():
    rng = np.random.default_rng(1)
    for (N, L, eps) in [(8, 2 * np.pi, 1e-7), (8, 2 * np.pi, 1e-6), (8, 2 * np.pi, 1e-3),
                        (8, 4 * np.pi, 1e-12), (16, 4 * np.pi, 1e-7)]:
        plan = pb.make_plan(N, L, eps)
        op = o.make_plan(N, L, eps)
        M = 2000
        pts = rng.random((M, 3)) * L
        pts[0] = 0
        pts[1] = [L - 1e-13, 0.5 * L, 1e-14]
        cr = rng.standard_normal(M)
        cc = cr + 1j * rng.standard_normal(M)
        f = rng.standard_normal((N,) * 3) + 1j * rng.standard_normal((N,) * 3)
        tag = f"N={N} eps={eps} w={plan.window.w}"
        stage(f"type1 real {tag}", lambda: rel(pb.type1(plan, pts, cr).coeffs, o.type1(op, pts, cr)))
        stage(f"type1 cplx {tag}", lambda: rel(pb.type1(plan, pts, cc).coeffs, o.type1(op, pts, cc)))
        stage(f"type2 {tag}", lambda: rel(pb.type2(plan, f, pts), o.type2(op, f, pts)))
        herm = [np.fft.fftshift(np.fft.fftn(rng.standard_normal((N,) * 3))) / N ** 3
                for _ in range(3)]
        stage(f"gather3 {tag}", lambda: rel(pb.nufft.gather3_real(plan, herm, pts),
                                            o.gather3_real(op, herm, pts)))
    # config-1 style step
    for kind in ("landau", "penning"):
        mk = pb.landau_spec if kind == "landau" else pb.penning_spec
        spec = mk(N=16, ppm=16, dt=0.05, steps=20, seed=0)
        ens = pb.sample_landau(spec, 0) if kind == "landau" else pb.sample_penning(spec, 0)
        plan = pb.make_plan(spec.N, spec.L, 1e-7)
        op = o.make_plan(spec.N, spec.L, 1e-7)
        rho_o = o.deposit_charge(ens.x, ens.q_per_particle, op)
        stage(f"{kind} deposit", lambda: rel(pb.deposit_charge(ens, plan).coeffs, rho_o))
        Eo = o.gather_efield(o.poisson_efield(rho_o, spec.L), ens.x, op)
        stage(f"{kind} gather", lambda: rel(
            pb.gather_efield(*pb.poisson_efield(pb.FourierField(16, spec.L, rho_o)), ens, plan), Eo))

        def run():
            setup = pb.RunSetup(spec=spec, eps=1e-7)
            res = pb.spawn_spmd(1, lambda ctx: pb.run_serial(setup, ctx))[0]
            got = np.array([[r.field_energy, r.kinetic_energy, r.total_energy]
                            for r in [res["initial"]] + res["records"]])
            ref = o.run_pd(op, ens.x, ens.v, ens.q_per_particle, ens.m_per_particle, L=spec.L,
                           B=spec.B_ext, e_kind=spec.e_kind, dt=spec.dt, steps=spec.steps)
            refa = np.array([[r[2], r[3], r[4]] for r in [ref["initial"]] + ref["records"]])
            return float(np.max(np.abs(got - refa) / np.abs(refa)))
        stage(f"{kind} 20-step trace max rel", run)


if __name__ == "__main__":
    main()
