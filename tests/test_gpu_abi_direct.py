"""Entry points of the C ABI that the Python API does not route through,
called directly (ctypes, device pointers) the way a reference-side binding
would, against the oracle."""

import ctypes

import numpy as np
import pytest

from conftest import oracle, rel_l2

import paper_2605_10729_b200 as pb
from paper_2605_10729_b200 import _native

pytestmark = pytest.mark.gpu


def _case(N=16, M=5000, seed=4):
    rng = np.random.default_rng(seed)
    plan = pb.make_plan(N, 2 * np.pi, 1e-7)
    x = rng.random((M, 3)) * plan.L
    c = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    f = rng.standard_normal((N,) * 3) + 1j * rng.standard_normal((N,) * 3)
    return plan, x, c, f


def test_pif_type1_complex_aos_points(cuda):
    """pif_type1_complex (AoS wrapped points, complex strengths; replaces
    spread_c + fftn, _kernels.py:31-54, nufft.py:132-145)."""
    torch = cuda
    o = oracle()
    plan, x, c, _ = _case()
    dp = plan.native("cuda")
    pts = torch.as_tensor(np.mod(x, plan.L), device="cuda")
    vals = torch.view_as_real(torch.as_tensor(c, device="cuda")).contiguous()
    modes = torch.empty((plan.N,) * 3, dtype=torch.complex128, device="cuda")
    _native.call("pif_type1_complex", dp.handle, pts.data_ptr(), vals.data_ptr(), x.shape[0],
                 modes.data_ptr(), _native.stream_handle())
    ref = o.type1(o.make_plan(plan.N, plan.L, 1e-7), x, c)
    assert rel_l2(modes.cpu().numpy(), ref) <= 1e-12


def test_pif_type2_complex_aos_points(cuda):
    """pif_type2_complex (replaces ifftn + interp_c, _kernels.py:99-122,
    nufft.py:159-172)."""
    torch = cuda
    o = oracle()
    plan, x, _, f = _case()
    dp = plan.native("cuda")
    pts = torch.as_tensor(np.mod(x, plan.L), device="cuda")
    fm = torch.as_tensor(f, device="cuda").contiguous()
    out = torch.empty(x.shape[0], dtype=torch.complex128, device="cuda")
    _native.call("pif_type2_complex", dp.handle, fm.data_ptr(), pts.data_ptr(), x.shape[0],
                 out.data_ptr(), _native.stream_handle())
    ref = o.type2(o.make_plan(plan.N, plan.L, 1e-7), f, x)
    assert rel_l2(out.cpu().numpy(), ref) <= 1e-12


def test_pif_poisson_and_field_energy(cuda):
    """pif_poisson (spectral.poisson_efield) and pif_field_energy
    (spectral.field_energy of poisson_efield) against the oracle."""
    torch = cuda
    o = oracle()
    plan, x, _, _ = _case()
    rho = o.deposit_charge(x, -0.01, o.make_plan(plan.N, plan.L, 1e-7))
    E = pb.poisson_efield(pb.FourierField(plan.N, plan.L, rho))
    Eo = o.poisson_efield(rho, plan.L)
    for a, b in zip(E, Eo):
        assert isinstance(a.coeffs, np.ndarray)
        assert np.array_equal(a.coeffs, b) or rel_l2(a.coeffs, b) <= 1e-15
    dp = plan.native("cuda")
    scalars = torch.zeros(4, dtype=torch.float64, device="cuda")
    r = torch.as_tensor(rho, device="cuda")
    _native.call("pif_field_energy", dp.handle, r.data_ptr(), scalars.data_ptr(),
                 _native.stream_handle())
    assert float(scalars[0]) == pytest.approx(o.field_energy(Eo, plan.L), rel=1e-13)
