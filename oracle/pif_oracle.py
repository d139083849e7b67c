"""CPU ORACLE — TEST INFRASTRUCTURE ONLY (parity checker and CPU baseline).

A numpy + C restatement of the reference's particle-decomposition PIF step
(/root/reference/pkg/src/pifsim).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this
module; the product package never does.

Pinning: ``tests/test_oracle.py`` checks every function here against golden
vectors produced by the reference itself (``tests/golden/make_golden.py``,
which imports /root/reference in the build container), plus the reference's
own known-answer tests (point at origin, constant field, direct sums).

Each function cites the reference file:line it restates.  The window kernels
run in C (``pif_oracle.c`` -> ``liboracle.so``, ctypes releases the GIL so
rank threads run in parallel, like the reference's nogil numba kernels).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading
import time
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_LIB_LOCK = threading.Lock()


def lib():
    """Load (building on first use) the C window kernels."""
    global _LIB
    with _LIB_LOCK:
        if _LIB is None:
            path = os.path.join(_HERE, "liboracle.so")
            src = os.path.join(_HERE, "pif_oracle.c")
            if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
                subprocess.run(["make", "-s", "-C", _HERE], check=True)
            L = ctypes.CDLL(path)
            dp = ctypes.POINTER(ctypes.c_double)
            i64 = ctypes.c_int64
            for name in ("oracle_spread_r", "oracle_spread_c"):
                fn = getattr(L, name)
                fn.argtypes = [dp, dp, dp, i64, i64, ctypes.c_double, ctypes.c_int, ctypes.c_double]
                fn.restype = None
            L.oracle_interp_c.argtypes = [dp, dp, dp, i64, i64, ctypes.c_double, ctypes.c_int,
                                          ctypes.c_double]
            L.oracle_interp_c.restype = None
            L.oracle_interp_r3.argtypes = [dp, dp, dp, dp, dp, i64, i64, ctypes.c_double,
                                           ctypes.c_int, ctypes.c_double]
            L.oracle_interp_r3.restype = None
            L.oracle_stencil.argtypes = [ctypes.c_double, i64, ctypes.c_int, ctypes.c_double, dp,
                                         ctypes.POINTER(i64)]
            L.oracle_stencil.restype = i64
            _LIB = L
    return _LIB


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


# ---------------------------------------------------------------------------
# Plan: nufft.py:66-102
# ---------------------------------------------------------------------------

@dataclass
class Plan:
    N: int
    L: float
    eps: float
    w: int
    beta: float
    n: int
    deconv: np.ndarray
    trunc: np.ndarray

    @property
    def h(self) -> float:
        return self.L / self.n


def mode_ints(N: int) -> np.ndarray:
    """spectral.py:33-35 — m = -N/2 .. N/2-1."""
    return np.arange(N) - N // 2


def window_transform(w: int, beta: float, n: int, N: int, L: float) -> np.ndarray:
    """nufft.py:87-102 — psi_hat(k_m) by 80-node Gauss-Legendre on [0, alpha]."""
    h = L / n
    alpha = 0.5 * w * h
    nodes, weights = np.polynomial.legendre.leggauss(80)
    u = 0.5 * (nodes + 1.0)
    gw = 0.5 * weights
    phi = np.exp(beta * (np.sqrt(np.maximum(1.0 - u * u, 0.0)) - 1.0))
    k = (2.0 * np.pi / L) * mode_ints(N)
    return (2.0 * alpha / L) * (np.cos(np.outer(k, alpha * u)) @ (gw * phi))


def make_plan(N: int, L: float, eps: float) -> Plan:
    """nufft.py:66-84 (validation at :72-77)."""
    if N % 2 != 0 or N < 4:
        raise ValueError(f"N must be even and >= 4, got {N}")
    if not (1e-16 <= eps <= 1e-1):
        raise ValueError(f"eps out of range: {eps}")
    if not (L > 0 and math.isfinite(L)):
        raise ValueError(f"invalid L {L}")
    w = math.ceil(abs(math.log10(eps)) - 1e-9) + 1
    beta = 2.30 * w
    n = math.ceil(2.0 * N)
    n += n % 2
    psi = window_transform(w, beta, n, N, L)
    return Plan(N, L, eps, w, beta, n, 1.0 / psi, mode_ints(N) % n)


# ---------------------------------------------------------------------------
# Transforms: nufft.py:105-189, 199-222
# ---------------------------------------------------------------------------

def prep_points(points: np.ndarray, L: float) -> np.ndarray:
    """nufft.py:105-113 — wrap into [0, L)."""
    w = np.mod(np.asarray(points, dtype=np.float64), L)
    w[w >= L] -= L
    return np.ascontiguousarray(w)


def spread_real(plan: Plan, pts: np.ndarray, vals: np.ndarray) -> np.ndarray:
    grid = np.zeros(plan.n ** 3)
    lib().oracle_spread_r(_p(pts), _p(np.ascontiguousarray(vals, dtype=np.float64)), _p(grid),
                          pts.shape[0], plan.n, plan.h, plan.w, plan.beta)
    return grid


def modes_from_grid(plan: Plan, grid: np.ndarray) -> np.ndarray:
    """nufft.py:140-145 — fftn, truncate to the mode block, deconvolve, 1/n^3."""
    n = plan.n
    spec = np.fft.fftn(grid.reshape(n, n, n))
    j = plan.trunc
    block = np.ascontiguousarray(spec[np.ix_(j, j, j)])
    d = plan.deconv
    block *= d[:, None, None]
    block *= d[None, :, None]
    block *= d[None, None, :]
    block *= 1.0 / n ** 3
    return block


def type1(plan: Plan, points: np.ndarray, strengths: np.ndarray) -> np.ndarray:
    """nufft.py:122-145."""
    pts = prep_points(points, plan.L)
    s = np.asarray(strengths)
    n = plan.n
    if np.isrealobj(s):
        grid = spread_real(plan, pts, s)
    else:
        sc = np.ascontiguousarray(s, dtype=np.complex128)
        g = np.zeros(2 * n ** 3)
        lib().oracle_spread_c(_p(pts), _p(sc.view(np.float64)), _p(g), pts.shape[0], n, plan.h,
                              plan.w, plan.beta)
        grid = g.view(np.complex128)
    return modes_from_grid(plan, grid)


def padded_spectrum(plan: Plan, coeffs: np.ndarray) -> np.ndarray:
    """nufft.py:148-156."""
    n = plan.n
    d = np.array(coeffs, dtype=np.complex128)
    dc = plan.deconv
    d *= dc[:, None, None]
    d *= dc[None, :, None]
    d *= dc[None, None, :]
    pad = np.zeros((n, n, n), dtype=np.complex128)
    j = plan.trunc
    pad[np.ix_(j, j, j)] = d
    return pad


def type2(plan: Plan, coeffs: np.ndarray, points: np.ndarray) -> np.ndarray:
    """nufft.py:159-172."""
    pts = prep_points(points, plan.L)
    u = np.ascontiguousarray(np.fft.ifftn(padded_spectrum(plan, coeffs)))
    out = np.empty(pts.shape[0], dtype=np.complex128)
    lib().oracle_interp_c(_p(pts), _p(u.view(np.float64).ravel()), _p(out.view(np.float64)),
                          pts.shape[0], plan.n, plan.h, plan.w, plan.beta)
    return out


def field_grids(plan: Plan, components) -> list:
    """nufft.py:182-185 — real parts of ifftn of each padded block."""
    return [np.ascontiguousarray(np.fft.ifftn(padded_spectrum(plan, c)).real).ravel()
            for c in components]


def interp3(plan: Plan, grids, pts: np.ndarray) -> np.ndarray:
    out = np.empty((pts.shape[0], 3))
    lib().oracle_interp_r3(_p(pts), _p(grids[0]), _p(grids[1]), _p(grids[2]), _p(out),
                           pts.shape[0], plan.n, plan.h, plan.w, plan.beta)
    return out


def gather3_real(plan: Plan, components, points: np.ndarray) -> np.ndarray:
    """nufft.py:175-189."""
    return interp3(plan, field_grids(plan, components), prep_points(points, plan.L))


def mode_matrix(N: int, L: float) -> np.ndarray:
    """spectral.py:38-44."""
    m = mode_ints(N)
    mx, my, mz = np.meshgrid(m, m, m, indexing="ij")
    return (2.0 * np.pi / L) * np.stack([mx.ravel(), my.ravel(), mz.ravel()], 1).astype(np.float64)


def direct_type1(plan: Plan, points, strengths) -> np.ndarray:
    """nufft.py:199-209 — exact sum F[k] = sum_j c_j exp(-i k.x_j)."""
    pts = prep_points(points, plan.L)
    s = np.asarray(strengths, dtype=np.complex128)
    K = mode_matrix(plan.N, plan.L)
    acc = np.zeros(K.shape[0], dtype=np.complex128)
    for lo in range(0, pts.shape[0], 2048):
        ch = pts[lo:lo + 2048]
        acc += np.exp(-1j * (ch @ K.T)).T @ s[lo:lo + ch.shape[0]]
    return acc.reshape(plan.N, plan.N, plan.N)


def direct_type2(plan: Plan, coeffs, points) -> np.ndarray:
    """nufft.py:212-222 — exact sum v_j = sum_k f_k exp(+i k.x_j)."""
    pts = prep_points(points, plan.L)
    K = mode_matrix(plan.N, plan.L)
    f = np.asarray(coeffs).ravel().astype(np.complex128)
    out = np.empty(pts.shape[0], dtype=np.complex128)
    for lo in range(0, pts.shape[0], 2048):
        ch = pts[lo:lo + 2048]
        out[lo:lo + ch.shape[0]] = np.exp(1j * (ch @ K.T)) @ f
    return out


# ---------------------------------------------------------------------------
# Spectral + cycle: spectral.py:57-101, pif.py:43-158, 240-245
# ---------------------------------------------------------------------------

def poisson_efield(rho: np.ndarray, L: float):
    """spectral.py:63-82."""
    N = rho.shape[0]
    k1 = (2.0 * np.pi / L) * mode_ints(N).astype(np.float64)
    kx, ky, kz = k1[:, None, None], k1[None, :, None], k1[None, None, :]
    k2 = kx * kx + ky * ky + kz * kz
    z = N // 2
    k2[z, z, z] = 1.0
    g = rho * (-1j / k2)
    out = [kx * g, ky * g, kz * g]
    for c in out:
        c[z, z, z] = 0.0
    return out


def field_energy(E, L: float) -> float:
    """spectral.py:85-91."""
    total = 0.0
    for f in E:
        c = f.ravel()
        total += np.vdot(c, c).real
    return 0.5 * L ** 3 * total


def hermitian_mismatch(coeffs: np.ndarray) -> float:
    """spectral.py:94-101."""
    a = coeffs[1:, 1:, 1:]
    b = coeffs[:0:-1, :0:-1, :0:-1]
    return 0.0 if a.size == 0 else float(np.max(np.abs(a - np.conj(b))))


def shape_factors(N: int, shape: str) -> np.ndarray:
    """pif.py:71-86."""
    if shape == "delta":
        return np.ones(N)
    if shape == "cic":
        m = np.arange(N) - N // 2
        u = np.pi * m / N
        s = np.ones(N)
        nz = m != 0
        s[nz] = (np.sin(u[nz]) / u[nz]) ** 2
        return s
    raise ValueError(shape)


def apply_shape(c: np.ndarray, s: np.ndarray) -> None:
    c *= s[:, None, None]
    c *= s[None, :, None]
    c *= s[None, None, :]


def finish_deposit(raw: np.ndarray, plan: Plan, shape: str = "delta") -> np.ndarray:
    """pif.py:95-105."""
    r = raw.copy()
    apply_shape(r, shape_factors(plan.N, shape))
    r *= 1.0 / plan.L ** 3
    m = plan.N // 2
    r[m, m, m] = 0.0
    return r


def deposit_charge(x: np.ndarray, q: float, plan: Plan, shape: str = "delta") -> np.ndarray:
    """pif.py:108-112."""
    return finish_deposit(type1(plan, x, np.full(x.shape[0], q)), plan, shape)


def gather_efield(E, x: np.ndarray, plan: Plan, shape: str = "delta") -> np.ndarray:
    """pif.py:115-137 (without the symmetry guard's exception type)."""
    s = shape_factors(plan.N, shape)
    comps = []
    for f in E:
        scale = np.max(np.abs(f))
        if scale > 0 and hermitian_mismatch(f) > 1e-10 * scale:
            raise ValueError("field lost Hermitian symmetry")
        c = f.copy()
        apply_shape(c, s)
        comps.append(c)
    return gather3_real(plan, comps, x)


def external_field(L: float, e_kind: str, x: np.ndarray) -> np.ndarray:
    """pif.py:43-57 — quadrupole (-15/L(x-L/2), -15/L(y-L/2), 30/L(z-L/2))."""
    if e_kind == "none":
        return np.zeros_like(x)
    c = L / 2.0
    out = np.empty_like(x)
    out[:, 0] = (-15.0 / L) * (x[:, 0] - c)
    out[:, 1] = (-15.0 / L) * (x[:, 1] - c)
    out[:, 2] = (30.0 / L) * (x[:, 2] - c)
    return out


def external_potential(L: float, e_kind: str, x: np.ndarray, q: float) -> float:
    """pif.py:60-68."""
    if e_kind == "none":
        return 0.0
    dx = x - L / 2.0
    phi = (7.5 / L) * (dx[:, 0] ** 2 + dx[:, 1] ** 2) - (15.0 / L) * dx[:, 2] ** 2
    return q * float(np.sum(phi))


def wrap(x: np.ndarray, L: float) -> np.ndarray:
    """particles.py:65-70."""
    w = np.mod(x, L)
    w[w >= L] -= L
    return w


def boris_push(x, v, E_at, q, m, B, e_kind, dt, L):
    """pif.py:140-158.  Returns new (x, v)."""
    qm = q / m
    E_tot = E_at + external_field(L, e_kind, x)
    half = 0.5 * dt * qm
    vm = v + half * E_tot
    Bv = np.asarray(B, dtype=np.float64)
    if np.any(Bv != 0.0):
        t = half * Bv
        s = 2.0 * t / (1.0 + t @ t)
        vp = vm + np.cross(vm, t)
        vm = vm + np.cross(vp, s)
    v = vm + half * E_tot
    return wrap(x + dt * v, L), v


# ---------------------------------------------------------------------------
# Particle-decomposition stepping loop: strategies.py:96-117, 148-173, 285-332
# ---------------------------------------------------------------------------

def tree_sum(arrays):
    """comm.py:329-339 — fixed binary-tree order."""
    level = list(arrays)
    while len(level) > 1:
        nxt = [level[i] + level[i + 1] for i in range(0, len(level) - 1, 2)]
        if len(level) % 2:
            nxt.append(level[-1])
        level = nxt
    return level[0]


def run_pd(plan: Plan, x: np.ndarray, v: np.ndarray, q: float, m: float, *, L: float,
           B=(0.0, 0.0, 0.0), e_kind="none", dt: float, steps: int, ranks: int = 1,
           shape: str = "delta", threads: bool = True, total_charge: float = 0.0,
           keep_first: bool = False):
    """Particle decomposition with `ranks` id slices (bench.py:184-188), each
    spread on its own thread, raw coefficients summed in fixed tree order.

    Returns dict(records=[(step, t, W, KE, total, px, py, pz, charge)],
    initial=record, x, v, rho0, E0) — rho0/E0 (first solve / first gather)
    only when keep_first.
    """
    M = x.shape[0]
    bounds = []
    base, extra = divmod(M, ranks)
    for r in range(ranks):
        lo = r * base + min(r, extra)
        bounds.append((lo, lo + base + (1 if r < extra else 0)))
    xs = [np.ascontiguousarray(x[lo:hi]) for lo, hi in bounds]
    vs = [np.ascontiguousarray(v[lo:hi]) for lo, hi in bounds]

    def par(fn):
        out = [None] * ranks
        if threads and ranks > 1:
            def run(r):
                out[r] = fn(r)
            ts = [threading.Thread(target=run, args=(r,)) for r in range(ranks)]
            for t in ts:
                t.start()
            for t in ts:
                t.join()
        else:
            for r in range(ranks):
                out[r] = fn(r)
        return out

    def solve():
        raws = par(lambda r: type1(plan, xs[r], np.full(xs[r].shape[0], q)))
        return finish_deposit(tree_sum(raws), plan, shape)

    def record(step, t, rho):
        def local(r):
            vv = vs[r]
            p = m * vv.sum(axis=0)
            return np.array([0.5 * m * float(np.sum(vv * vv)), p[0], p[1], p[2],
                             external_potential(L, e_kind, xs[r], q), 0.0])
        tot = tree_sum(par(local))
        W = field_energy(poisson_efield(rho, L), L)
        ke, px, py, pz, u = tot[:5]
        return (step, t, W, ke, W + ke + u, px, py, pz, total_charge)

    out = {}
    rho = solve()
    if keep_first:
        out["rho0"] = rho.copy()
    initial = record(0, 0.0, rho)
    records = []
    for i in range(steps):
        E = poisson_efield(rho, L)
        s = shape_factors(plan.N, shape)
        comps = []
        for f in E:
            c = f.copy()
            apply_shape(c, s)
            comps.append(c)
        grids = field_grids(plan, comps)
        E_at = par(lambda r: interp3(plan, grids, prep_points(xs[r], L)))
        if keep_first and i == 0:
            out["E0"] = np.concatenate(E_at, axis=0)
        for r in range(ranks):
            xs[r], vs[r] = boris_push(xs[r], vs[r], E_at[r], q, m, B, e_kind, dt, L)
        rho = solve()
        records.append(record(i + 1, (i + 1) * dt, rho))
    out.update(records=records, initial=initial, x=np.concatenate(xs), v=np.concatenate(vs))
    return out


class PDRun:
    """Stateful oracle PD stepper for timing (bench.py cpu_baseline and
    --impl reference): `ranks` id slices on `ranks` threads, like the
    reference's spawn_spmd PD run (strategies.py:285-303).

    ``phase_s`` accumulates wall seconds per phase so the bench can report the
    split between the particle kernels (spread, interp, push: linear in the
    particle count) and the mode-space work (per-rank fftn + truncate, 3 x
    ifftn of the padded spectra: fixed per step for a given N)."""

    PHASES = ("spread", "fftn", "field_grids", "interp", "push")

    def __init__(self, plan: Plan, x, v, q, m, *, L, B=(0.0, 0.0, 0.0), e_kind="none", dt,
                 ranks=1, shape="delta"):
        self.plan, self.q, self.m, self.L, self.B = plan, q, m, L, B
        self.e_kind, self.dt, self.ranks, self.shape = e_kind, dt, ranks, shape
        M = x.shape[0]
        base, extra = divmod(M, ranks)
        self.xs, self.vs = [], []
        for r in range(ranks):
            lo = r * base + min(r, extra)
            hi = lo + base + (1 if r < extra else 0)
            self.xs.append(np.ascontiguousarray(x[lo:hi]))
            self.vs.append(np.ascontiguousarray(v[lo:hi]))
        self.phase_s = dict.fromkeys(self.PHASES, 0.0)
        self.rho = self._solve()

    def _par(self, fn):
        out = [None] * self.ranks
        ts = [threading.Thread(target=lambda r=r: out.__setitem__(r, fn(r)))
              for r in range(self.ranks)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        return out

    def _timed(self, phase, fn):
        t0 = time.perf_counter()
        out = fn()
        self.phase_s[phase] += time.perf_counter() - t0
        return out

    def _solve(self):
        # type1 per rank (nufft.py:122-145), split into its spread and its
        # fftn + truncate so the two can be timed apart
        plan = self.plan
        grids = self._timed("spread", lambda: self._par(lambda r: spread_real(
            plan, prep_points(self.xs[r], self.L), np.full(self.xs[r].shape[0], self.q))))
        raws = self._timed("fftn", lambda: self._par(lambda r: modes_from_grid(plan, grids[r])))
        return finish_deposit(tree_sum(raws), plan, self.shape)

    def step(self):
        plan = self.plan
        E = poisson_efield(self.rho, self.L)
        s = shape_factors(plan.N, self.shape)
        comps = []
        for f in E:
            c = f.copy()
            apply_shape(c, s)
            comps.append(c)
        grids = self._timed("field_grids", lambda: field_grids(plan, comps))
        E_at = self._timed("interp", lambda: self._par(
            lambda r: interp3(plan, grids, prep_points(self.xs[r], self.L))))

        def push(r):
            # each rank thread pushes its own slice, as the reference's rank
            # threads do (numpy releases the GIL inside the array kernels)
            self.xs[r], self.vs[r] = boris_push(self.xs[r], self.vs[r], E_at[r], self.q,
                                                self.m, self.B, self.e_kind, self.dt, self.L)
        self._timed("push", lambda: self._par(push))
        self.rho = self._solve()
        return field_energy(poisson_efield(self.rho, self.L), self.L)
