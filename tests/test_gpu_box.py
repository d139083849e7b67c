"""Box-mode (sparse-set) kernels against the column kernels and the oracle.

Below ~12 particles per stencil cell the engine bins particles by 8^3-cell
boxes (key_of, box layout) and runs spread_box_kernel / interp_box_kernel:
one CTA per box with the box's footprint in shared memory.  PIF_BOX=0/1
(read at plan creation) forces the layout, so the same inputs go through both
kernel families here; both must match the oracle (oracle/, pinned to the
reference's golden vectors) and the reference's own traces.
"""

import ctypes

import numpy as np
import pytest

from conftest import golden, oracle, rel_l2

import paper_2605_10729_b200 as pb
from paper_2605_10729_b200 import _native

pytestmark = pytest.mark.gpu

TIGHT = 1e-12


@pytest.fixture(params=["0", "1"], ids=["columns", "boxes"])
def layout(request, monkeypatch):
    monkeypatch.setenv("PIF_BOX", request.param)
    return request.param


def _engine_state(kind, N, M, shape="delta"):
    import torch
    from paper_2605_10729_b200.engine import PifEngine
    mk = pb.landau_spec if kind == "landau" else pb.penning_spec
    spec = mk(N=N, ppm=max(1, M // N ** 3), dt=0.003125, seed=0)
    q, m = spec.Q_e / spec.num_particles, abs(spec.Q_e) / spec.num_particles
    plan = pb.make_plan(N, spec.L, 1e-7)
    eng = PifEngine(plan, spec.num_particles, "cuda", q=q, m=m, externals=spec.externals(),
                    dt=spec.dt, shape=shape)
    eng.load_sampled(spec, (0, spec.num_particles))
    x0, v0 = (t.cpu().numpy() for t in eng.to_id_order())
    eng.particle_diag()
    eng.deposit()
    eng.solve_fields()
    rho = eng.rho.cpu().numpy()
    E = torch.empty((eng.count, 3), dtype=torch.float64, device="cuda")
    cur = eng._soa()
    _native.call("pif_interp_perm", eng.handle, ctypes.byref(cur), eng.parts.perm.data_ptr(),
                 E.data_ptr(), _native.stream_handle())
    eng.interp_push()
    x1, v1 = (t.cpu().numpy() for t in eng.to_id_order())
    diag = eng.diag.cpu().numpy()
    eng.rebin()
    eng.deposit()
    eng.solve_fields()
    rho1 = eng.rho.cpu().numpy()
    return dict(spec=spec, plan=plan, x0=x0, v0=v0, rho=rho, E=E.cpu().numpy(), x1=x1, v1=v1,
                diag=diag, rho1=rho1, q=q, m=m, layout=_native.load().pif_key_layout(eng.handle))


CASES = [("landau", 64, 1 << 21), ("landau", 128, 1 << 22), ("penning", 64, 1 << 22)]


@pytest.mark.parametrize("kind,N,M", CASES, ids=[f"{k}-{N}-2p{M.bit_length() - 1}"
                                                  for k, N, M in CASES])
def test_sparse_step_matches_oracle_in_both_layouts(kind, N, M, layout):
    o = oracle()
    st = _engine_state(kind, N, M)
    assert st["layout"] == int(layout)
    spec, plan = st["spec"], st["plan"]
    op = o.make_plan(N, spec.L, 1e-7)
    rho_o = o.deposit_charge(st["x0"], st["q"], op)
    assert rel_l2(st["rho"], rho_o) <= TIGHT
    sel = np.sort(np.random.default_rng(3).choice(spec.num_particles, 8192, replace=False))
    E_o = o.gather_efield(o.poisson_efield(rho_o, spec.L), st["x0"][sel], op)
    assert rel_l2(st["E"][sel], E_o) <= TIGHT
    x1o, v1o = o.boris_push(st["x0"][sel], st["v0"][sel], E_o, st["q"], st["m"], spec.B_ext,
                            spec.e_kind, spec.dt, spec.L)
    assert rel_l2(st["v1"][sel], v1o) <= TIGHT
    dx = np.abs(st["x1"][sel] - x1o)
    assert float(np.minimum(dx, spec.L - dx).max()) <= 1e-12 * spec.L
    assert st["diag"][0] == pytest.approx(float(np.sum(st["v1"] ** 2)), rel=1e-12)
    rho1_o = o.deposit_charge(st["x1"], st["q"], op)
    assert rel_l2(st["rho1"], rho1_o) <= TIGHT


def test_layouts_agree_to_rounding(monkeypatch):
    out = {}
    for lay in ("0", "1"):
        monkeypatch.setenv("PIF_BOX", lay)
        out[lay] = _engine_state("landau", 64, 1 << 21)
    for k in ("rho", "E", "v1", "rho1"):
        assert rel_l2(out["1"][k], out["0"][k]) <= 1e-13, k


@pytest.mark.parametrize("kind,dt", [("landau", 0.05), ("penning", 0.05)])
def test_config1_traces_in_both_layouts(kind, dt, layout):
    spec = (pb.landau_spec if kind == "landau" else pb.penning_spec)(N=16, ppm=16, dt=dt,
                                                                      steps=20, seed=0)
    res = pb.spawn_spmd(1, lambda ctx: pb.run_serial(pb.RunSetup(spec=spec, eps=1e-7), ctx))[0]
    got = np.array([[r.field_energy, r.kinetic_energy, r.total_energy]
                    for r in [res["initial"]] + res["records"]])
    ref = golden("config1.npz")[f"{kind}_trace"][:, 2:5]
    assert np.max(np.abs(got - ref) / np.abs(ref)) <= 1e-10


def test_operator_api_in_box_layout(layout):
    """type1 (real and complex strengths) and type2 through SortedPoints +
    the box kernels, against the oracle."""
    o = oracle()
    rng = np.random.default_rng(11)
    plan = pb.make_plan(32, 2 * np.pi, 1e-7)
    op = o.make_plan(32, 2 * np.pi, 1e-7)
    x = rng.random((40000, 3)) * plan.L
    c = rng.standard_normal(40000)
    cc = c + 1j * rng.standard_normal(40000)
    assert rel_l2(pb.type1(plan, x, c).coeffs, o.type1(op, x, c)) <= TIGHT
    assert rel_l2(pb.type1(plan, x, cc).coeffs, o.type1(op, x, cc)) <= TIGHT
    f = rng.standard_normal((32,) * 3) + 1j * rng.standard_normal((32,) * 3)
    assert rel_l2(pb.type2(plan, f, x), o.type2(op, f, x)) <= TIGHT
