"""Seeded random configurations through every kernel family (DMMA w <= 8 with
FMA tail sub-batches, FMA ring w = 9..14, one-thread-per-particle, complex
strengths) against the oracle: grid size, tolerance, density and clustering
drawn per case."""

import numpy as np
import pytest

from conftest import oracle, rel_l2

import paper_2605_10729_b200 as pb
from paper_2605_10729_b200 import nufft

pytestmark = pytest.mark.gpu

TIGHT = 1e-12


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    N = int(rng.choice([4, 6, 8, 10, 12, 16, 24]))
    eps = float(rng.choice([1e-1, 1e-2, 1e-3, 1e-5, 1e-7, 1e-9, 1e-12, 1e-14, 1e-15, 1e-16]))
    M = int(rng.integers(1, 20000))
    L = float(rng.choice([1.0, 2 * np.pi, 25.0]))
    if rng.random() < 0.5:
        x = rng.random((M, 3)) * L
    else:                                   # clustered, some points outside [0, L)
        x = L / 2 + rng.standard_normal((M, 3)) * L * rng.uniform(0.02, 0.3)
    return rng, N, eps, M, L, x


@pytest.mark.parametrize("seed", range(40))
def test_random_configuration_matches_oracle(seed):
    o = oracle()
    rng, N, eps, M, L, x = _case(seed)
    plan, op = pb.make_plan(N, L, eps), o.make_plan(N, L, eps)
    q = rng.standard_normal(M)
    got = pb.type1(plan, x, q).coeffs
    assert rel_l2(got, o.type1(op, x, q)) <= TIGHT, (N, eps, M)
    c = q + 1j * rng.standard_normal(M)
    assert rel_l2(pb.type1(plan, x, c).coeffs, o.type1(op, x, c)) <= TIGHT, (N, eps, M)
    herm = [np.fft.fftshift(np.fft.fftn(rng.standard_normal((N,) * 3))) / N ** 3
            for _ in range(3)]
    assert rel_l2(nufft.gather3_real(plan, herm, x), o.gather3_real(op, herm, x)) <= TIGHT
    f = rng.standard_normal((N,) * 3) + 1j * rng.standard_normal((N,) * 3)
    assert rel_l2(pb.type2(plan, f, x), o.type2(op, f, x)) <= TIGHT, (N, eps, M)


@pytest.mark.parametrize("seed", range(12))
def test_random_engine_step_matches_oracle(seed):
    """One PIF step (deposit, Poisson, gather + Boris push with random B and the
    quadrupole or no external E) on a random configuration."""
    from conftest import rel_max
    o = oracle()
    rng, N, eps, M, L, x = _case(500 + seed)
    x = np.mod(x, L)
    v = rng.standard_normal((M, 3))
    B = tuple(float(b) for b in rng.uniform(-5, 5, 3)) if rng.random() < 0.5 else (0.0, 0.0, 0.0)
    e_kind = "quadrupole" if rng.random() < 0.5 else "none"
    q, m, dt = -1.0 / M, 1.0 / M, float(rng.choice([0.003125, 0.05]))
    plan, op = pb.make_plan(N, L, eps), o.make_plan(N, L, eps)
    ens = pb.ParticleEnsemble(x=x.copy(), v=v.copy(), ids=np.arange(M), q_per_particle=q,
                              m_per_particle=m, total_charge=q * M, total_mass=m * M,
                              global_count=M)
    st = pb.pif_step(pb.StepState(ensemble=ens, plan=plan, dt=dt,
                                  externals=pb.ExternalFieldsSpec(L=L, B=B, e_kind=e_kind)))
    rho = o.deposit_charge(x, q, op)
    Eo = o.gather_efield(o.poisson_efield(rho, L), x, op)
    xo, vo = o.boris_push(x.copy(), v.copy(), Eo, q, m, B, e_kind, dt, L)
    assert rel_max(st.ensemble.v, vo) <= 1e-11, (N, eps, M)
    dx = np.abs(st.ensemble.x - xo)
    assert np.max(np.minimum(dx, L - dx)) <= 1e-11 * L, (N, eps, M)


@pytest.mark.parametrize("seed", range(6))
def test_random_pd_run_matches_serial(seed):
    """PD over 1-3 thread ranks equals the serial run on random small specs."""
    rng = np.random.default_rng(2000 + seed)
    mk = pb.landau_spec if rng.random() < 0.5 else pb.penning_spec
    spec = mk(N=int(rng.choice([4, 8, 12])), ppm=int(rng.integers(1, 6)),
              dt=float(rng.choice([0.003125, 0.05])), steps=int(rng.integers(1, 12)),
              seed=int(rng.integers(0, 5)))
    setup = pb.RunSetup(spec=spec, eps=float(rng.choice([1e-5, 1e-7, 1e-10])))
    ref = pb.spawn_spmd(1, lambda ctx: pb.run_serial(setup, ctx))[0]
    ranks = int(rng.integers(2, 4))
    got = pb.spawn_spmd(ranks, lambda ctx: pb.run_particle_decomposition(setup, ctx))[0]
    a = np.array([r.total_energy for r in ref["records"]])
    b = np.array([r.total_energy for r in got["records"]])
    assert np.max(np.abs(a - b) / np.abs(a)) <= 1e-10


@pytest.mark.parametrize("seed", range(6))
def test_random_device_sampler_matches_host(seed):
    """The device Philox samplers regenerate the host (reference) ensemble for
    random specs, seeds and id slices."""
    from paper_2605_10729_b200.samplers import sample_benchmark, sample_device
    rng = np.random.default_rng(3000 + seed)
    mk = pb.landau_spec if rng.random() < 0.5 else pb.penning_spec
    spec = mk(N=int(rng.choice([4, 8, 12])), ppm=int(rng.integers(1, 30)),
              seed=int(rng.integers(0, 1000)))
    n = spec.num_particles
    lo = int(rng.integers(0, n))
    hi = int(rng.integers(lo, n + 1))
    host = sample_benchmark(spec, spec.seed, (lo, hi))
    x, v, ids = sample_device(spec, (lo, hi), "cuda")
    assert np.array_equal(ids.cpu().numpy(), host.ids)
    if hi > lo:
        assert np.max(np.abs(x.cpu().numpy() - host.x)) <= 1e-10 * spec.L
        assert np.max(np.abs(v.cpu().numpy() - host.v)) <= 1e-12
