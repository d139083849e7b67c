"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py) and against the reference's own known answers.
CPU only."""

import numpy as np
import pytest

from conftest import golden, oracle, rel_l2, rel_max

CASES = golden("nufft_cases.npz")
NCASE = len({k.split("_")[0] for k in CASES.files})


def _plan(ci):
    N, L, eps = CASES[f"c{ci}_meta"]
    return oracle().make_plan(int(N), float(L), float(eps))


@pytest.mark.parametrize("ci", range(NCASE))
def test_plan_tables_match_reference(ci):
    plan = _plan(ci)
    assert np.array_equal(plan.deconv, CASES[f"c{ci}_deconv"])


@pytest.mark.parametrize("ci", range(NCASE))
def test_type1_real_matches_reference(ci):
    got = oracle().type1(_plan(ci), CASES[f"c{ci}_pts"], CASES[f"c{ci}_cr"])
    assert rel_max(got, CASES[f"c{ci}_t1_real"]) <= 1e-14


@pytest.mark.parametrize("ci", range(NCASE))
def test_type1_complex_matches_reference(ci):
    got = oracle().type1(_plan(ci), CASES[f"c{ci}_pts"], CASES[f"c{ci}_cc"])
    assert rel_max(got, CASES[f"c{ci}_t1_cplx"]) <= 1e-14


@pytest.mark.parametrize("ci", range(NCASE))
def test_type2_matches_reference(ci):
    got = oracle().type2(_plan(ci), CASES[f"c{ci}_f"], CASES[f"c{ci}_pts"])
    assert rel_max(got, CASES[f"c{ci}_t2"]) <= 1e-14


@pytest.mark.parametrize("ci", range(NCASE))
def test_gather3_matches_reference(ci):
    comps = [CASES[f"c{ci}_herm{d}"] for d in range(3)]
    got = oracle().gather3_real(_plan(ci), comps, CASES[f"c{ci}_pts"])
    assert rel_max(got, CASES[f"c{ci}_g3"]) <= 1e-14


@pytest.mark.parametrize("ci", [i for i in range(NCASE) if f"c{i}_d1" in CASES.files])
def test_direct_sums_match_reference(ci):
    o = oracle()
    plan = _plan(ci)
    assert rel_max(o.direct_type1(plan, CASES[f"c{ci}_pts"], CASES[f"c{ci}_cc"]),
                   CASES[f"c{ci}_d1"]) <= 1e-13
    assert rel_max(o.direct_type2(plan, CASES[f"c{ci}_f"], CASES[f"c{ci}_pts"]),
                   CASES[f"c{ci}_d2"]) <= 1e-13


@pytest.mark.parametrize("ci", range(NCASE))
def test_nufft_accuracy_vs_direct(ci):
    # the reference's own accuracy bar: <= 10 eps vs direct sums (test_nufft.py:62-69)
    o = oracle()
    plan = _plan(ci)
    if plan.N > 8:
        pytest.skip("direct sums kept small")
    pts, cc, f = CASES[f"c{ci}_pts"], CASES[f"c{ci}_cc"], CASES[f"c{ci}_f"]
    assert rel_max(o.type1(plan, pts, cc), o.direct_type1(plan, pts, cc)) <= 10 * plan.eps
    assert rel_max(o.type2(plan, f, pts), o.direct_type2(plan, f, pts)) <= 10 * plan.eps


def test_known_answers():
    o = oracle()
    plan = o.make_plan(8, 2 * np.pi, 1e-7)
    F = o.type1(plan, np.zeros((1, 3)), np.ones(1))          # test_nufft.py:50-53
    assert np.max(np.abs(F - 1.0)) <= 10 * plan.eps
    assert np.all(o.type1(plan, np.zeros((0, 3)), np.zeros(0)) == 0)
    N = plan.N
    f = np.zeros((N,) * 3, complex)
    f[N // 2, N // 2, N // 2] = 2.5 - 0.5j                    # test_nufft.py:92-100
    pts = np.random.default_rng(13).random((20, 3)) * plan.L
    assert np.max(np.abs(o.type2(plan, f, pts) - (2.5 - 0.5j))) <= 10 * plan.eps * 2.6


CFG = golden("config1.npz")


@pytest.fixture(scope="module")
def ensembles():
    from paper_2605_10729_b200.samplers import landau_spec, penning_spec, sample_benchmark
    out = {}
    for kind, mk in (("landau", landau_spec), ("penning", penning_spec)):
        spec = mk(N=16, ppm=16, dt=0.05, steps=20, seed=0)
        out[kind] = (spec, sample_benchmark(spec, 0))
    return out


@pytest.mark.parametrize("kind", ["landau", "penning"])
def test_oracle_first_step_matches_reference(kind, ensembles):
    o = oracle()
    spec, ens = ensembles[kind]
    plan = o.make_plan(spec.N, spec.L, 1e-7)
    rho = o.deposit_charge(ens.x, ens.q_per_particle, plan)
    assert rel_l2(rho, CFG[f"{kind}_rho0"]) <= 1e-14
    E = o.gather_efield(o.poisson_efield(rho, spec.L), ens.x, plan)
    sel = np.arange(0, ens.count, 16)
    assert rel_l2(E[sel], CFG[f"{kind}_E0_sel"]) <= 1e-13
    x1, v1 = o.boris_push(ens.x, ens.v, E, ens.q_per_particle, ens.m_per_particle, spec.B_ext,
                          spec.e_kind, spec.dt, spec.L)
    assert rel_l2(v1[sel], CFG[f"{kind}_v1_sel"]) <= 1e-13
    assert np.max(np.abs(x1[sel] - CFG[f"{kind}_x1_sel"])) <= 1e-12 * spec.L


@pytest.mark.parametrize("kind,dt,tag,ranks", [("landau", 0.05, "", 1),
                                               ("penning", 0.05, "", 1),
                                               ("landau", 0.05, "_pd2", 2)])
def test_oracle_trace_matches_reference(kind, dt, tag, ranks):
    from paper_2605_10729_b200.samplers import landau_spec, penning_spec, sample_benchmark
    o = oracle()
    mk = landau_spec if kind == "landau" else penning_spec
    spec = mk(N=16, ppm=16, dt=dt, steps=20, seed=0)
    ens = sample_benchmark(spec, 0)
    plan = o.make_plan(spec.N, spec.L, 1e-7)
    res = o.run_pd(plan, ens.x, ens.v, ens.q_per_particle, ens.m_per_particle, L=spec.L,
                   B=spec.B_ext, e_kind=spec.e_kind, dt=dt, steps=20, ranks=ranks,
                   total_charge=spec.Q_e)
    got = np.array([res["initial"]] + res["records"])
    ref = CFG[f"{kind}{tag}_trace"]
    for col in (2, 3, 4):   # field, kinetic, total energy
        assert np.max(np.abs(got[:, col] - ref[:, col]) / np.abs(ref[:, col])) <= 1e-12
