"""The particle-in-Fourier cycle (deposit, Poisson, gather, Boris push).

Same public API as the reference's ``pifsim.pif`` (/root/reference/pkg/src/pifsim/pif.py)
for the PIF path: ``ExternalFieldsSpec``, ``external_field_eval``,
``external_potential_energy``, ``shape_factors``, ``finish_deposit``,
``deposit_charge``, ``gather_efield``, ``boris_push``, ``StepState``,
``pif_step``, ``kinetic_energy``, ``momentum``.  The heavy parts run on the
B200: deposit = binned sm_100a spreading + cuFFT (csrc/particles.cu,
csrc/fields.cu); gather = fused padded spectra + batched Z2D + register-tiled
interpolation; the push is the same device code the fused interp+push kernel
uses.  The FFT-PIC coarse stepper (pif.py:197-237) belongs to the parareal
strategy and is out of scope here.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native, nufft
from ._device import as_device, is_torch, like_input, require_cuda
from .diag import NULL_TIMERS
from .particles import ParticleEnsemble, wrap_positions
from .spectral import FourierField, hermitian_mismatch, poisson_efield


class FieldSymmetryError(RuntimeError):
    """Gather input lost the Hermitian pairing a real field must carry."""


@dataclass(frozen=True)
class ExternalFieldsSpec:
    """Constant magnetic field plus an optional quadrupole electric field
    (pif.py:27-37)."""

    L: float
    B: tuple = (0.0, 0.0, 0.0)
    e_kind: str = "none"

    def __post_init__(self):
        if self.e_kind not in ("none", "quadrupole"):
            raise ValueError(f"unknown external E-field kind {self.e_kind!r}")


NO_EXTERNALS = ExternalFieldsSpec(L=1.0)


def external_field_eval(spec: ExternalFieldsSpec, x):
    """(-15/L (x-L/2), -15/L (y-L/2), +30/L (z-L/2)) or zeros (pif.py:43-57)."""
    if is_torch(x):
        import torch
        if spec.e_kind == "none":
            return torch.zeros_like(x)
        c = spec.L / 2.0
        return torch.stack([(-15.0 / spec.L) * (x[:, 0] - c), (-15.0 / spec.L) * (x[:, 1] - c),
                            (30.0 / spec.L) * (x[:, 2] - c)], dim=1)
    x = np.asarray(x, dtype=np.float64)
    if spec.e_kind == "none":
        return np.zeros_like(x)
    c = spec.L / 2.0
    out = np.empty_like(x)
    out[:, 0] = (-15.0 / spec.L) * (x[:, 0] - c)
    out[:, 1] = (-15.0 / spec.L) * (x[:, 1] - c)
    out[:, 2] = (30.0 / spec.L) * (x[:, 2] - c)
    return out


def external_potential_energy(spec: ExternalFieldsSpec, ens: ParticleEnsemble) -> float:
    """q * sum phi_ext(x) (pif.py:60-68)."""
    if spec.e_kind == "none":
        return 0.0
    c = spec.L / 2.0
    dx = ens.x - c
    phi = (7.5 / spec.L) * (dx[:, 0] ** 2 + dx[:, 1] ** 2) - (15.0 / spec.L) * dx[:, 2] ** 2
    return ens.q_per_particle * float(phi.sum())


def shape_factors(plan: nufft.NufftPlan, shape: str) -> np.ndarray:
    """Per-dimension particle shape transform S_k (pif.py:71-86)."""
    if shape == "delta":
        return np.ones(plan.N)
    if shape == "cic":
        return nufft._cic_factors(plan.N)
    raise ValueError(f"unknown shape {shape!r}")


def _apply_shape(coeffs, s: np.ndarray):
    if is_torch(coeffs):
        import torch
        st = torch.as_tensor(s, device=coeffs.device)
        coeffs *= st[:, None, None]
        coeffs *= st[None, :, None]
        coeffs *= st[None, None, :]
    else:
        coeffs *= s[:, None, None]
        coeffs *= s[None, :, None]
        coeffs *= s[None, None, :]


def finish_deposit(f: FourierField, plan: nufft.NufftPlan, shape: str = "delta") -> FourierField:
    """Shape transform, 1/L^3, zero k=0 (pif.py:95-105)."""
    _apply_shape(f.coeffs, shape_factors(plan, shape))
    f.coeffs *= 1.0 / plan.L ** 3
    mid = plan.N // 2
    f.coeffs[mid, mid, mid] = 0.0
    f.units = "charge-density"
    return f


def deposit_charge(ens: ParticleEnsemble, plan: nufft.NufftPlan,
                   shape: str = "delta") -> FourierField:
    """rho_k = (S_k / L^3) sum_j q_j exp(-i k.x_j) (pif.py:108-112)."""
    if is_torch(ens.x):
        import torch
        strengths = torch.full((ens.count,), ens.q_per_particle, dtype=torch.float64,
                               device=ens.x.device)
    else:
        strengths = np.full(ens.count, ens.q_per_particle)
    return finish_deposit(nufft.type1(plan, ens.x, strengths), plan, shape)


def gather_efield(Ex: FourierField, Ey: FourierField, Ez: FourierField, ens: ParticleEnsemble,
                  plan: nufft.NufftPlan, shape: str = "delta"):
    """E(x_j) = sum_k E_k S_k exp(+i k.x_j), (M, 3) (pif.py:115-137).

    Raises FieldSymmetryError when a component's Hermitian pairing is broken
    beyond 1e-10 of its scale (checked on the device, pif.py:128-133)."""
    E, scalars = nufft.gather_fields_at(plan, (Ex, Ey, Ez), ens.x, shape)
    worst = float(scalars[1])
    if worst > 1e-10:
        for f in (Ex, Ey, Ez):
            c = as_device(f.coeffs, complex_=True)
            scale = float(c.abs().max())
            mm = hermitian_mismatch(c)
            if scale > 0 and mm > 1e-10 * scale:
                raise FieldSymmetryError(
                    f"{f.units} modes lost Hermitian symmetry "
                    f"(mismatch {mm:.3e} vs scale {scale:.3e})")
    return like_input(E, ens.x)


def boris_constants(qm: float, dt: float, B):
    """half = 0.5 dt q/m, t = half B, s = 2t/(1+t.t) as numpy computes them
    (pif.py:146-153)."""
    half = 0.5 * dt * qm
    Bv = np.asarray(B, dtype=np.float64)
    has_b = bool(np.any(Bv != 0.0))
    t = half * Bv
    s = 2.0 * t / (1.0 + t @ t) if has_b else np.zeros(3)
    return half, t, s, has_b


def boris_push(ens: ParticleEnsemble, E_at, externals: ExternalFieldsSpec, dt: float,
               L: float) -> ParticleEnsemble:
    """Boris scheme with periodic wrap; mutates and returns the ensemble
    (pif.py:140-158).  Runs as torch ops on the device (the hot-path push is
    fused into the interp kernel, csrc/particles.cu boris_one)."""
    if tuple(E_at.shape) != tuple(ens.x.shape):
        raise ValueError(f"E_at shape {tuple(E_at.shape)} does not match particles")
    torch = require_cuda()
    qm = ens.q_per_particle / ens.m_per_particle
    half, t, s, has_b = boris_constants(qm, dt, externals.B)
    x = as_device(ens.x)
    v = as_device(ens.v, device=x.device)
    E = as_device(E_at, device=x.device)
    E_tot = E + external_field_eval(externals, x)
    vm = v + half * E_tot
    if has_b:
        tt = torch.as_tensor(t, device=x.device)
        ss = torch.as_tensor(s, device=x.device)
        vp = vm + torch.linalg.cross(vm, tt.expand_as(vm))
        vm = vm + torch.linalg.cross(vp, ss.expand_as(vp))
    v = vm + half * E_tot
    x = wrap_positions(x + dt * v, L)
    ens.x = like_input(x, ens.x)
    ens.v = like_input(v, ens.v)
    return ens


@dataclass
class StepState:
    """Everything one rank needs to advance its particles one step (pif.py:161-175)."""

    ensemble: ParticleEnsemble
    plan: nufft.NufftPlan
    externals: ExternalFieldsSpec
    dt: float
    t: float = 0.0
    step: int = 0
    shape: str = "delta"

    def __post_init__(self):
        if self.dt <= 0:
            raise ValueError(f"dt must be positive, got {self.dt}")


def pif_step(state: StepState, timers=NULL_TIMERS) -> StepState:
    """One PIF cycle (pif.py:178-190): deposit, Poisson, gather, push — on the
    device through the fused engine (one spread, one field solve, one fused
    interp+push launch).  The engine (native plan, cuFFT plans, grids, SoA
    store) is created once per (plan, device, particle count) and reused by
    later calls; raises FieldSymmetryError when the gathered field modes lost
    their Hermitian pairing, as gather_efield does (pif.py:128-133)."""
    from ._device import default_device
    from .engine import PifEngine
    ens = state.ensemble
    eng = PifEngine.cached(state.plan, ens.count, default_device(ens.x), q=ens.q_per_particle,
                           m=ens.m_per_particle, externals=state.externals, dt=state.dt,
                           shape=state.shape)
    with timers.section("Scatter"):
        eng.load(ens.x, ens.v)
        eng.deposit()
    with timers.section("Gather"):
        eng.solve_fields()
        guard = float(eng.scalars[1])
        if guard > 1e-10:
            raise FieldSymmetryError(f"field modes lost Hermitian symmetry (relative mismatch "
                                     f"{guard:.3e})")
    with timers.section("ParticleUpdate"):
        eng.gather_push()
    eng.store_into(ens)
    state.t += state.dt
    state.step += 1
    return state


def kinetic_energy(ens: ParticleEnsemble) -> float:
    return 0.5 * ens.m_per_particle * float((ens.v * ens.v).sum())


def momentum(ens: ParticleEnsemble):
    v = ens.v
    if is_torch(v):
        return ens.m_per_particle * v.sum(dim=0).cpu().numpy()
    return ens.m_per_particle * v.sum(axis=0)
