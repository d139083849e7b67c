"""Generate golden fixtures from the REFERENCE implementation itself.

Run in the build container only (the reference does not exist on GPU boxes):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Writes tests/golden/*.npz.  Every array here is produced by calling pifsim's
public API (nufft.type1/type2/gather3_real, pif.deposit_charge/gather_efield/
boris_push, strategies.run_serial/run_particle_decomposition, diag.fit_damping_rate)
on seeded inputs; the tests compare the CPU oracle and the CUDA path against them.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

OUT = os.path.dirname(os.path.abspath(__file__))


def _pifsim():
    try:
        import pifsim  # noqa: F401
    except ImportError:
        sys.path.insert(0, "/root/reference/pkg/src")
    import pifsim
    return pifsim


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def nufft_cases(pifsim):
    from pifsim import nufft
    rng = np.random.default_rng(2605)
    out = {}
    cases = [(8, 1e-3), (8, 1e-6), (8, 1e-7), (8, 1e-12), (16, 1e-7), (12, 1e-7)]
    for ci, (N, eps) in enumerate(cases):
        L = 2 * np.pi if ci % 2 == 0 else 4 * np.pi
        plan = nufft.make_plan(N, L, eps)
        M = 300
        pts = rng.random((M, 3)) * L
        pts[0] = 0.0                       # point at origin
        pts[1] = [L - 1e-13, 0.5 * L, 1e-14]  # near the periodic seam
        pts[2] = [-0.25 * L, 1.5 * L, 0.3]    # needs wrapping
        cr = rng.standard_normal(M)
        cc = rng.standard_normal(M) + 1j * rng.standard_normal(M)
        f = rng.standard_normal((N,) * 3) + 1j * rng.standard_normal((N,) * 3)
        herm = [np.fft.fftshift(np.fft.fftn(rng.standard_normal((N,) * 3))) / N ** 3
                for _ in range(3)]
        p = f"c{ci}_"
        out[p + "meta"] = np.array([N, L, eps])
        out[p + "deconv"] = plan.deconv
        out[p + "pts"] = pts
        out[p + "cr"] = cr
        out[p + "cc"] = cc
        out[p + "f"] = f
        out[p + "t1_real"] = nufft.type1(plan, pts, cr).coeffs
        out[p + "t1_cplx"] = nufft.type1(plan, pts, cc).coeffs
        out[p + "t2"] = nufft.type2(plan, f, pts)
        for d in range(3):
            out[p + f"herm{d}"] = herm[d]
        out[p + "g3"] = nufft.gather3_real(plan, herm, pts)
        if N <= 8:
            out[p + "d1"] = nufft.direct_type1(plan, pts, cc).coeffs
            out[p + "d2"] = nufft.direct_type2(plan, f, pts)
    return out


def config1(pifsim, kind: str, dt: float, steps: int, ranks: int = 1, tag: str = ""):
    from pifsim import nufft, pif
    from pifsim.bench import landau_spec, penning_spec, sample_benchmark
    from pifsim.comm import spawn_spmd
    from pifsim.spectral import poisson_efield
    from pifsim.strategies import RunSetup, run_particle_decomposition, run_serial
    mk = landau_spec if kind == "landau" else penning_spec
    spec = mk(N=16, ppm=16, dt=dt, steps=steps, seed=0)
    setup = RunSetup(spec=spec, eps=1e-7)
    out = {}
    p = f"{kind}{tag}_"
    if ranks == 1:
        ens = sample_benchmark(spec, spec.seed)
        out[p + "sha_xv"] = np.frombuffer(sha(ens.x, ens.v).encode(), dtype=np.uint8)
        plan = nufft.make_plan(spec.N, spec.L, 1e-7)
        rho = pif.deposit_charge(ens, plan)
        out[p + "rho0"] = rho.coeffs
        E = pif.gather_efield(*poisson_efield(rho), ens, plan)
        sel = np.arange(0, ens.count, 16)
        out[p + "E0_sel"] = E[sel]
        out[p + "E0_norm"] = np.array([np.linalg.norm(E)])
        e2 = ens.copy()
        pif.boris_push(e2, E, spec.externals(), dt, spec.L)
        out[p + "x1_sel"] = e2.x[sel]
        out[p + "v1_sel"] = e2.v[sel]
        res = spawn_spmd(1, lambda ctx: run_serial(setup, ctx))[0]
    else:
        res = spawn_spmd(ranks, lambda ctx: run_particle_decomposition(setup, ctx))[0]
    recs = [res["initial"]] + res["records"]
    cols = ("step", "t", "field_energy", "kinetic_energy", "total_energy", "px", "py", "pz",
            "total_charge")
    out[p + "trace"] = np.array([[getattr(r, c) for c in cols] for r in recs])
    return out


def damping(pifsim):
    from pifsim.comm import spawn_spmd
    from pifsim.bench import landau_spec
    from pifsim.diag import fit_damping_rate
    from pifsim.strategies import RunSetup, run_serial
    spec = landau_spec(N=16, ppm=10, dt=0.05, steps=200, seed=0)
    res = spawn_spmd(1, lambda ctx: run_serial(RunSetup(spec=spec, eps=1e-7), ctx))[0]
    t = np.array([r.t for r in res["records"]])
    w = np.array([r.field_energy for r in res["records"]])
    return {"damp_t": t, "damp_w": w, "damp_gamma": np.array([fit_damping_rate(t, w)])}


def sampler_hashes(pifsim):
    from pifsim.bench import landau_spec, penning_spec, sample_benchmark
    out = {}
    for kind, mk in (("landau", landau_spec), ("penning", penning_spec)):
        for (N, ppm, seed) in ((8, 4, 2), (16, 16, 0), (8, 3, 7)):
            spec = mk(N=N, ppm=ppm, seed=seed)
            e = sample_benchmark(spec, seed)
            out[f"sampler_{kind}_{N}_{ppm}_{seed}"] = np.frombuffer(
                sha(e.x, e.v, e.ids).encode(), dtype=np.uint8)
    return out


def main():
    pifsim = _pifsim()
    np.savez_compressed(os.path.join(OUT, "nufft_cases.npz"), **nufft_cases(pifsim))
    cfg = {}
    cfg.update(config1(pifsim, "landau", 0.05, 20))
    cfg.update(config1(pifsim, "landau", 0.003125, 20, tag="_slow"))
    cfg.update(config1(pifsim, "penning", 0.05, 20))
    cfg.update(config1(pifsim, "landau", 0.05, 20, ranks=2, tag="_pd2"))
    np.savez_compressed(os.path.join(OUT, "config1.npz"), **cfg)
    np.savez_compressed(os.path.join(OUT, "damping.npz"), **damping(pifsim))
    np.savez_compressed(os.path.join(OUT, "samplers.npz"), **sampler_hashes(pifsim))
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
