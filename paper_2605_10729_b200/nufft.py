"""Type-1 / type-2 NUFFTs on a periodic box, B200 edition.

API mirrors the reference's ``pifsim.nufft`` shared-memory part
(/root/reference/pkg/src/pifsim/nufft.py:32-231):

    type 1:  F[k] = sum_j c_j exp(-i k.x_j)          (points -> modes)
    type 2:  v_j  = sum_k f_k exp(+i k.x_j)            (modes -> points)

with the same exponential-of-semicircle window (w = ceil(|log10 eps|)+1,
sigma = 2, beta = 2.30 w), the same Gauss-Legendre window transform and the same
fine-grid layout, so results match the reference to rounding.  The host plan
below computes every constant with numpy exactly as nufft.py:66-102 does and
hands them to the device plan (libpifb200, include/pif_b200.h), which owns the
cuFFT plans and buffers.  Spreading / gathering run in the sm_100a kernels of
csrc/particles.cu; the slab (domain-decomposition) variants are out of scope.
"""

from __future__ import annotations

import math
import threading
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _native
from ._device import as_device, default_device, is_torch, like_input, require_cuda
from .spectral import FourierField, mode_ints, mode_matrix, wavenumber_vector


@dataclass(frozen=True)
class WindowSpec:
    w: int
    sigma: float
    beta: float

    def __post_init__(self):
        if self.w < 2 or self.sigma < 1.25 or self.beta <= 0:
            raise ValueError(f"invalid window: {self}")


class DevicePlan:
    """Owner of one native plan (cuFFT plans, fine grid, spectra, field grid,
    cell tables) on one CUDA device."""

    def __init__(self, plan: "NufftPlan", device_index: int):
        lib = _native.load()
        N = plan.N
        self._tables = [np.ascontiguousarray(plan.deconv, dtype=np.float64),
                        np.ascontiguousarray(wavenumber_vector(N, plan.L)),
                        np.ascontiguousarray(_cic_factors(N))]
        d = _native.pif_plan_desc_t(
            N, float(plan.L), float(plan.eps), int(plan.window.w), float(plan.window.beta),
            int(plan.n_up), self._tables[0].ctypes.data, self._tables[1].ctypes.data,
            self._tables[2].ctypes.data, 1.0 / plan.L ** 3, 0.5 * plan.L ** 3)
        handle = _native.ctypes.c_void_p()
        _native.check(lib.pif_plan_create(_native.ctypes.byref(d), int(device_index),
                                          _native.ctypes.byref(handle)), "pif_plan_create")
        self.handle = handle.value
        self.device_index = int(device_index)
        self._fin = weakref.finalize(self, lib.pif_plan_destroy, handle.value)

    @property
    def device_bytes(self) -> int:
        return int(_native.load().pif_plan_device_bytes(self.handle))

    def close(self):
        self._fin()


def _cic_factors(N: int) -> np.ndarray:
    """Cloud-in-cell S_k on the mode set (pif.py:79-85)."""
    m = np.arange(N) - N // 2
    u = np.pi * m / N
    s = np.ones(N)
    nz = m != 0
    s[nz] = (np.sin(u[nz]) / u[nz]) ** 2
    return s


@dataclass(eq=False)
class NufftPlan:
    N: int
    L: float
    eps: float
    window: WindowSpec
    n_up: int
    deconv: np.ndarray = field(init=False)
    _trunc: np.ndarray = field(init=False)

    def __post_init__(self):
        psi_hat = _window_transform(self.window, self.n_up, self.N, self.L)
        if not np.all(np.isfinite(psi_hat)) or np.any(psi_hat <= 0):
            raise ValueError("window transform must be strictly positive over the band")
        self.deconv = 1.0 / psi_hat
        self._trunc = np.asarray(mode_ints(self.N) % self.n_up)
        self._native: dict[int, DevicePlan] = {}
        self._lock = threading.Lock()

    @property
    def h(self) -> float:
        return self.L / self.n_up

    def native(self, device=None) -> DevicePlan:
        """Device plan on `device` (created on first use, one per device)."""
        torch = require_cuda()
        dev = torch.device(device) if device is not None else default_device()
        idx = dev.index if dev.index is not None else torch.cuda.current_device()
        with self._lock:
            dp = self._native.get(idx)
            if dp is None:
                dp = DevicePlan(self, idx)
                self._native[idx] = dp
        return dp


def make_plan(N: int, L: float, eps: float) -> NufftPlan:
    """Plan for N modes per dimension at tolerance eps (nufft.py:66-84)."""
    if N % 2 != 0 or N < 4:
        raise ValueError(f"N must be even and >= 4, got {N}")
    if not (1e-16 <= eps <= 1e-1):
        raise ValueError(f"eps out of range [1e-16, 1e-1]: {eps}")
    if not (L > 0 and math.isfinite(L)):
        raise ValueError(f"invalid domain length {L}")
    w = math.ceil(abs(math.log10(eps)) - 1e-9) + 1
    sigma = 2.0
    n_up = math.ceil(sigma * N)
    n_up += n_up % 2
    return NufftPlan(N=N, L=L, eps=eps, window=WindowSpec(w=w, sigma=sigma, beta=2.30 * w),
                     n_up=n_up)


def _window_transform(window: WindowSpec, n_up: int, N: int, L: float) -> np.ndarray:
    """psi_hat(k_m) by 80-node Gauss-Legendre on [0, alpha] (nufft.py:87-102)."""
    h = L / n_up
    alpha = 0.5 * window.w * h
    nodes, weights = np.polynomial.legendre.leggauss(80)
    u = 0.5 * (nodes + 1.0)
    gw = 0.5 * weights
    phi = np.exp(window.beta * (np.sqrt(np.maximum(1.0 - u * u, 0.0)) - 1.0))
    k = (2.0 * np.pi / L) * mode_ints(N)
    return (2.0 * alpha / L) * (np.cos(np.outer(k, alpha * u)) @ (gw * phi))


# ---------------------------------------------------------------------------
# argument handling (nufft.py:105-113, 124-129, 161-166)
# ---------------------------------------------------------------------------

def _points_device(points):
    torch = require_cuda()
    shape = tuple(points.shape) if hasattr(points, "shape") else np.asarray(points).shape
    if len(shape) != 2 or shape[1] != 3:
        raise ValueError(f"points must be (M, 3), got {shape}")
    pts = as_device(points)
    if pts.numel() and not bool(torch.isfinite(pts).all()):
        raise ValueError("non-finite point coordinates")
    return pts


class SortedPoints:
    """Arbitrary API points binned into ES-stencil cell order on the device.

    x, y, z are wrapped into [0, L) (nufft.py:105-113); ids record the input
    order so results can be written back per point."""

    def __init__(self, plan: NufftPlan, pts):
        torch = require_cuda()
        dp = plan.native(pts.device)
        M = int(pts.shape[0])
        self.count = M
        self.dp = dp
        dev = pts.device
        src = pts.t().contiguous().clone()          # (3, M) SoA copy
        ids = torch.arange(M, dtype=torch.int64, device=dev)
        stream = _native.stream_handle(dev)
        self.sorted = torch.empty((3, max(M, 1)), dtype=torch.float64, device=dev)
        self.ids = torch.empty(max(M, 1), dtype=torch.int64, device=dev)
        if M:
            _native.call("pif_wrap_points", dp.handle, src[0].data_ptr(), src[1].data_ptr(),
                         src[2].data_ptr(), M, stream)
            key = torch.empty(M, dtype=torch.int32, device=dev)
            rank = torch.empty(M, dtype=torch.int32, device=dev)
            s_src = _native.soa(src[0], src[1], src[2], ids=ids, count=M)
            _native.call("pif_bin_keys", dp.handle, _native.ctypes.byref(s_src),
                         key.data_ptr(), rank.data_ptr(), stream)
            s_dst = _native.soa(self.sorted[0], self.sorted[1], self.sorted[2], ids=self.ids,
                                count=M)
            _native.call("pif_bin_scatter", dp.handle, _native.ctypes.byref(s_src),
                         _native.ctypes.byref(s_dst), key.data_ptr(), rank.data_ptr(), 0, stream)
        self.view = _native.soa(self.sorted[0], self.sorted[1], self.sorted[2], ids=self.ids,
                                count=M)


def _wrapped_aos(plan: NufftPlan, pts):
    """Wrapped copy of (M,3) device points, AoS (complex-strength paths)."""
    torch = require_cuda()
    M = int(pts.shape[0])
    soa = pts.t().contiguous().clone()
    if M:
        _native.call("pif_wrap_points", plan.native(pts.device).handle, soa[0].data_ptr(),
                     soa[1].data_ptr(), soa[2].data_ptr(), M, _native.stream_handle(pts.device))
    return soa.t().contiguous()


def _is_real(s) -> bool:
    if is_torch(s):
        return not s.is_complex()
    return np.isrealobj(s)


def type1(plan: NufftPlan, points, strengths) -> FourierField:
    """Nonuniform points -> Fourier modes to O(eps) (nufft.py:122-145)."""
    torch = require_cuda()
    pts = _points_device(points)
    M = int(pts.shape[0])
    s_shape = tuple(strengths.shape) if hasattr(strengths, "shape") else np.shape(strengths)
    if s_shape != (M,):
        raise ValueError(f"strengths shape {s_shape} does not match {M} points")
    real = _is_real(strengths)
    s = as_device(strengths, complex_=not real, device=pts.device)
    if M and not bool(torch.isfinite(torch.view_as_real(s) if not real else s).all()):
        raise ValueError("non-finite strengths")
    dp = plan.native(pts.device)
    N = plan.N
    modes = torch.empty((N, N, N), dtype=torch.complex128, device=pts.device)
    stream = _native.stream_handle(pts.device)
    if real:
        sp = SortedPoints(plan, pts)
        _native.call("pif_spread_sorted", dp.handle, _native.ctypes.byref(sp.view),
                     s.data_ptr(), 0.0, stream)
        _native.call("pif_grid_to_modes", dp.handle, modes.data_ptr(), stream)
    else:
        sp = SortedPoints(plan, pts)
        s_re, s_im = s.real.contiguous(), s.imag.contiguous()
        _native.call("pif_type1_complex_sorted", dp.handle, _native.ctypes.byref(sp.view),
                     s_re.data_ptr(), s_im.data_ptr(), modes.data_ptr(), stream)
    return FourierField(N, plan.L, like_input(modes, points))


def _coeffs_of(plan: NufftPlan, modes):
    coeffs = modes.coeffs if isinstance(modes, FourierField) else modes
    shape = tuple(coeffs.shape)
    if shape != (plan.N, plan.N, plan.N):
        raise ValueError(f"modes shape {shape} does not match N={plan.N}")
    c = as_device(coeffs, complex_=True)
    import torch
    if not bool(torch.isfinite(torch.view_as_real(c)).all()):
        raise ValueError("non-finite mode coefficients")
    return c


def type2(plan: NufftPlan, modes, points):
    """Fourier modes -> values at nonuniform points to O(eps) (nufft.py:159-172)."""
    torch = require_cuda()
    c = _coeffs_of(plan, modes)
    pts = _points_device(points).to(c.device)
    M = int(pts.shape[0])
    if M == 0:
        return like_input(torch.empty(0, dtype=torch.complex128, device=c.device), points)
    E = torch.zeros((M, 3), dtype=torch.float64, device=c.device)
    sp = SortedPoints(plan, pts)
    _native.call("pif_type2_complex_sorted", plan.native(c.device).handle, c.data_ptr(),
                 _native.ctypes.byref(sp.view), E.data_ptr(), _native.stream_handle(c.device))
    out = torch.complex(E[:, 0].contiguous(), E[:, 1].contiguous())
    return like_input(out, points)


def gather_fields_at(plan: NufftPlan, comps, points, shape: str = "delta"):
    """Load three E-mode blocks into the plan's field grid (shape applied on the
    device) and gather them at the points; returns (E (M,3) device, guard)."""
    torch = require_cuda()
    cs = [as_device(c.coeffs if isinstance(c, FourierField) else c, complex_=True)
          for c in comps]
    for c in cs:
        if tuple(c.shape) != (plan.N,) * 3:
            raise ValueError(f"modes shape {tuple(c.shape)} does not match N={plan.N}")
    dev = cs[0].device
    pts = _points_device(points).to(dev)
    dp = plan.native(dev)
    stream = _native.stream_handle(dev)
    scalars = torch.zeros(4, dtype=torch.float64, device=dev)
    _native.call("pif_fields_from_modes", dp.handle, cs[0].data_ptr(), cs[1].data_ptr(),
                 cs[2].data_ptr(), _native.SHAPE[shape], scalars.data_ptr(), stream)
    M = int(pts.shape[0])
    E = torch.zeros((M, 3), dtype=torch.float64, device=dev)
    if M:
        sp = SortedPoints(plan, pts)
        _native.call("pif_interp_sorted", dp.handle, _native.ctypes.byref(sp.view),
                     E.data_ptr(), stream)
    return E, scalars


def gather3_real(plan: NufftPlan, components, points):
    """Fused type-2 of three real fields at the points, (M, 3) (nufft.py:175-189)."""
    E, _ = gather_fields_at(plan, components, points, "delta")
    return like_input(E, points)


# ---------------------------------------------------------------------------
# direct-sum transforms of the reference API (nufft.py:199-231), computed on the GPU
# ---------------------------------------------------------------------------

_DIRECT_CHUNK = 2048


def direct_type1(plan: NufftPlan, points, strengths) -> FourierField:
    torch = require_cuda()
    pts = _points_device(points)
    pts = torch.remainder(pts, plan.L)
    pts = torch.where(pts >= plan.L, pts - plan.L, pts)
    s = as_device(strengths, complex_=True, device=pts.device)
    K = torch.as_tensor(mode_matrix(plan.N, plan.L), device=pts.device)
    acc = torch.zeros(K.shape[0], dtype=torch.complex128, device=pts.device)
    for lo in range(0, pts.shape[0], _DIRECT_CHUNK):
        ch = pts[lo:lo + _DIRECT_CHUNK]
        acc += torch.exp(-1j * (ch @ K.T)).T @ s[lo:lo + ch.shape[0]]
    return FourierField(plan.N, plan.L, like_input(acc.reshape((plan.N,) * 3), points))


def direct_type2(plan: NufftPlan, modes, points):
    torch = require_cuda()
    coeffs = modes.coeffs if isinstance(modes, FourierField) else modes
    f = as_device(coeffs, complex_=True).reshape(-1)
    pts = _points_device(points).to(f.device)
    pts = torch.remainder(pts, plan.L)
    pts = torch.where(pts >= plan.L, pts - plan.L, pts)
    K = torch.as_tensor(mode_matrix(plan.N, plan.L), device=f.device)
    out = torch.empty(pts.shape[0], dtype=torch.complex128, device=f.device)
    for lo in range(0, pts.shape[0], _DIRECT_CHUNK):
        ch = pts[lo:lo + _DIRECT_CHUNK]
        out[lo:lo + ch.shape[0]] = torch.exp(1j * (ch @ K.T)) @ f
    return like_input(out, points)


def direct_transform(plan: NufftPlan, direction: str, *args):
    if direction == "type1":
        return direct_type1(plan, *args)
    if direction == "type2":
        return direct_type2(plan, *args)
    raise ValueError(f"direction must be 'type1' or 'type2', got {direction!r}")
