"""The reference's field-operator plugin point, backed by the B200 path.

The reference's stepping loop (/root/reference/pkg/src/pifsim/strategies.py:285-303
``_stepping_loop``) talks to its fields through a duck-typed protocol with three
methods, implemented there by ``_PifFieldOps`` (strategies.py:148-173):

    solve(ens)            -> FourierField   type-1 deposit, allreduce of the raw
                                            modes over the comm, finish_deposit
    gather(fields, ens)   -> (M, 3) float   Poisson solve + type-2 gather of E
    field_energy(fields)  -> float          (L^3/2) sum |E_k|^2 of that solve

``B200FieldOps`` is that object for the B200 build.  A reference user swaps one
constructor (``_PifFieldOps(plan, shape, comm, timers)`` ->
``B200FieldOps(plan, shape, comm, timers)``) and keeps the loop, the Recorder
and the Boris push.  Behind it sits one cached ``PifEngine`` per (plan,
device, particle count): ``solve`` uploads the positions, bins, spreads,
runs D2Z + truncate, allreduces the raw modes (in place on the device when
``comm`` is this package's ``Comm``; through the numpy ``allreduce_sum`` of any
other comm object), then runs the fused finish_deposit + Poisson + energy +
Hermitian guard + padded Z2D solve once.  ``gather`` and ``field_energy`` on
the fields ``solve`` returned reuse that solve (the loop always calls them on
the fields of the latest solve); fields from anywhere else are solved again
from their modes.
"""

from __future__ import annotations

import numpy as np

from . import _native
from ._device import as_device, default_device, is_torch, like_input, require_cuda
from .diag import NULL_TIMERS
from .spectral import FourierField

_NONE = object()


class B200FieldOps:
    """Replicated-mode PIF solve/gather on the GPU (strategies.py:148-173)."""

    def __init__(self, plan, shape: str = "delta", comm=None, timers=None, device=None):
        from .pif import ExternalFieldsSpec
        if shape not in _native.SHAPE:
            raise ValueError(f"unknown shape {shape!r}")
        self.plan = plan
        self.shape = shape
        self.comm = comm
        self.timers = timers if timers is not None else NULL_TIMERS
        self.device = device
        self._ext = ExternalFieldsSpec(L=plan.L)
        self._eng = None
        self._fields = _NONE        # the FourierField the engine's field grid holds
        self._x = _NONE             # the position array the engine's particles hold

    # -- engine ------------------------------------------------------------------
    def _engine(self, ens):
        from .engine import PifEngine
        dev = self.device if self.device is not None else default_device(ens.x)
        eng = PifEngine.cached(self.plan, ens.count, dev, q=ens.q_per_particle,
                               m=ens.m_per_particle, externals=self._ext, dt=1.0,
                               shape=self.shape)
        if eng is not self._eng:
            self._eng, self._fields, self._x = eng, _NONE, _NONE
        return eng

    def _load_positions(self, eng, ens):
        """Positions only (no velocities: nothing here pushes), wrapped and
        binned; ids 0..M-1 so gathered E comes back in ensemble order."""
        if self._x is ens.x:
            return
        eng.load(ens.x)
        self._x = ens.x

    def _allreduce(self, eng):
        c = self.comm
        if c is None or c.size == 1:
            return
        from .comm import Comm
        if isinstance(c, Comm):
            c.allreduce_sum(eng.raw)              # in place, on the device (NCCL)
        else:                                     # any allreduce_sum(numpy) comm object
            N3 = self.plan.N ** 3
            host = eng.raw.view(N3 * 2).cpu().numpy().view(np.complex128)
            tot = np.asarray(c.allreduce_sum(host), dtype=np.complex128)
            eng.raw.copy_(as_device(tot.view(np.float64), device=eng.device))

    # -- protocol ------------------------------------------------------------------
    def solve(self, ens) -> FourierField:
        """rho_k: type-1 deposit + allreduce + finish_deposit (strategies.py:155-164)."""
        eng = self._engine(ens)
        with self.timers.section("Scatter"):
            self._load_positions(eng, ens)
            eng.deposit()
        if self.comm is not None:
            with self.timers.section("Allreduce"):
                self._allreduce(eng)
        eng.solve_fields()
        rho = FourierField(self.plan.N, self.plan.L, like_input(eng.rho.clone(), ens.x),
                           "charge-density")
        self._fields = rho
        return rho

    def gather(self, rho: FourierField, ens):
        """E at the particles, (M, 3) like ens.x (strategies.py:166-170); raises
        FieldSymmetryError like gather_efield (pif.py:128-133)."""
        from .pif import FieldSymmetryError
        if tuple(ens.x.shape) != (ens.count, 3):
            raise ValueError(f"particles must be (M, 3), got {tuple(ens.x.shape)}")
        eng = self._engine(ens)
        torch = require_cuda()
        with self.timers.section("Gather"):
            if rho is not self._fields:
                self._solve_from(eng, rho)
            guard = float(eng.scalars[1])
            if guard > 1e-10:
                raise FieldSymmetryError(f"{rho.units} modes lost Hermitian symmetry "
                                         f"(relative mismatch {guard:.3e})")
            self._load_positions(eng, ens)
            E = torch.empty((ens.count, 3), dtype=torch.float64, device=eng.device)
            if ens.count:
                cur = eng._soa()
                _native.call("pif_interp_perm", eng.handle, _native.ctypes.byref(cur),
                             eng.parts.perm.data_ptr(), E.data_ptr(), eng._stream())
            return like_input(E, ens.x)

    def field_energy(self, rho: FourierField) -> float:
        """(L^3/2) sum |E_k|^2 of poisson_efield(rho) (strategies.py:172-173)."""
        if rho is self._fields and self._eng is not None:
            return float(self._eng.scalars[0])
        from .spectral import field_energy, poisson_efield
        return field_energy(*poisson_efield(rho))

    def _solve_from(self, eng, rho: FourierField):
        """Field grid of arbitrary rho modes, as gather_efield builds it:
        poisson_efield, then shape + padded spectra + Z2D + guard on the device
        (pif_fields_from_modes)."""
        from .spectral import poisson_efield
        if rho.N != self.plan.N:
            raise ValueError(f"modes N={rho.N} do not match the plan's N={self.plan.N}")
        dev_rho = FourierField(rho.N, rho.L, as_device(rho.coeffs, complex_=True,
                                                      device=eng.device), rho.units)
        E = [f.coeffs for f in poisson_efield(dev_rho)]
        _native.call("pif_field_energy", eng.handle, dev_rho.coeffs.data_ptr(),
                     eng.scalars.data_ptr(), eng._stream())
        _native.call("pif_fields_from_modes", eng.handle, E[0].data_ptr(), E[1].data_ptr(),
                     E[2].data_ptr(), _native.SHAPE[self.shape], eng.scalars.data_ptr(),
                     eng._stream())
        self._fields = rho


def field_ops(plan, shape="delta", comm=None, timers=None):
    """Factory with _PifFieldOps' argument order (strategies.py:152-156)."""
    return B200FieldOps(plan, shape, comm, timers)


__all__ = ["B200FieldOps", "field_ops"]
