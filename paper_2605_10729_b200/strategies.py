"""Serial and particle-decomposition runners (the north-star path).

Same entry points and return contract as the reference's strategies module
(/root/reference/pkg/src/pifsim/strategies.py:310-346): particles split into
contiguous id slices (bench.py:184-188), modes replicated on every rank, one
allreduce per step, per-step ``StepRecord`` diagnostics on the root rank.  The
whole step runs on the rank's GPU through ``engine.PifEngine``; the only host
work per run is sampling the initial ensemble and reading the records back.

Domain decomposition and the space-time (parareal) strategy are out of scope
for this tier: their runners exist for API compatibility and raise.
"""

from __future__ import annotations

import time as _time
from dataclasses import dataclass, field

import numpy as np

from . import nufft
from ._device import require_cuda
from .comm import Comm, RankContext
from .diag import StepRecord, Timers
from .engine import PifEngine
from .samplers import BenchmarkSpec, id_slice, sample_benchmark


@dataclass(frozen=True)
class RunSetup:
    """Resolved numerical configuration for one run (strategies.py:41-48)."""

    spec: BenchmarkSpec
    eps: float = 1e-7
    shape: str = "delta"
    diag_every: int = 1
    # "host": the reference's numpy sampler (bit-identical ensembles);
    # "device": the same streams regenerated in HBM (pif_sample_*, equal to
    # libm ulps); "auto": device above 2^22 particles, where the reference's
    # per-rank materialisation of the global ensemble stops fitting host memory
    sampler: str = "auto"
    # bit-reproducible stepping (stable binning + fixed-order plane reduction,
    # PifEngine.set_deterministic): the reference's runs are bit-identical by
    # construction (test_strategies.py:57-62, 405-409); off by default, the
    # atomic spread is the fast path
    deterministic: bool = False


@dataclass(frozen=True)
class CoarseSpec:
    kind: str = "pif"
    eps: float = 1e-3
    n_c: int | None = None
    dt: float | None = None

    def __post_init__(self):
        if self.kind not in ("pif", "pic"):
            raise ValueError(f"coarse kind must be pif|pic, got {self.kind!r}")


@dataclass(frozen=True)
class PararealConfig:
    ranks_time: int
    tol: float = 1e-8
    max_iters: int = 50
    coarse: CoarseSpec = field(default_factory=CoarseSpec)
    blocks: int = 1
    record_states: bool = False
    exact_iters: int | None = None


def records_from_table(table: np.ndarray, *, steps: int, dt: float, q: float, m: float,
                       total_charge: float, diag_every: int = 1):
    """Turn the device record table [W, sum v.v, sum v, sum phi, guard] into
    StepRecords exactly as Recorder.record composes them (strategies.py:96-117,
    pif.py:60-68, 240-245)."""
    every = max(1, diag_every)
    out = []
    for step in range(steps + 1):
        if step != 0 and step % every != 0:
            continue
        W, svv, sx, sy, sz, sphi = (float(a) for a in table[step, :6])
        ke = 0.5 * m * svv
        u_ext = q * sphi
        out.append(StepRecord(step=step, t=step * dt if step else 0.0, field_energy=W,
                              kinetic_energy=ke, total_energy=W + ke + u_ext, px=m * sx,
                              py=m * sy, pz=m * sz, total_charge=total_charge))
    return out


def _run_replicated(setup: RunSetup, comm: Comm | None, timers: Timers | None,
                    device=None) -> dict:
    """timers=None: no section timing, the steps replay from CUDA graphs;
    a Timers: synchronised wall-clock sections (the reference's semantics)."""
    torch = require_cuda()
    spec = setup.spec
    plan = nufft.make_plan(spec.N, spec.L, setup.eps)
    externals = spec.externals()
    size = comm.size if comm is not None else 1
    rank = comm.rank if comm is not None else 0
    lo, hi = id_slice(spec.num_particles, rank, size)
    n_p = spec.num_particles
    q, m = spec.Q_e / n_p, abs(spec.Q_e) / n_p        # bench.py:194-201
    if setup.sampler not in ("auto", "host", "device"):
        raise ValueError(f"unknown sampler {setup.sampler!r}")
    on_device = setup.sampler == "device" or (setup.sampler == "auto" and n_p > (1 << 22))
    dev = torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())
    with torch.cuda.device(dev):
        eng = PifEngine(plan, hi - lo, dev, q=q, m=m, externals=externals, dt=spec.dt,
                        shape=setup.shape, comm=comm,
                        deterministic=True if setup.deterministic else None)
        if on_device:
            eng.load_sampled(spec, (lo, hi))
        else:
            ens = sample_benchmark(spec, spec.seed, (lo, hi))
            eng.load(ens.x, ens.v, ens.ids)
        torch.cuda.synchronize(dev)
        start = _time.perf_counter()
        table = eng.run(spec.steps, timers=timers)
        host = table.cpu().numpy()
        loop_seconds = _time.perf_counter() - start
    # the guard ran on the device every step (pif.py:128-133); the run is not
    # stopped mid-graph, so report the first offending step as the reference
    # would have raised there
    bad = np.nonzero(host[:, 6] > 1e-10)[0] if host.size else []
    if len(bad):
        from .pif import FieldSymmetryError
        first = int(bad[0])
        raise FieldSymmetryError(f"field modes lost Hermitian symmetry at step {first} "
                                 f"(relative mismatch {float(host[first, 6]):.3e})")
    recs = records_from_table(host, steps=spec.steps, dt=spec.dt, q=q, m=m,
                              total_charge=spec.Q_e, diag_every=setup.diag_every)
    initial, records = recs[0], recs[1:]
    # the reference's Recorder stamps t = (i+1)*dt for step i+1 (strategies.py:301)
    for r in records:
        r.t = r.step * spec.dt
    return {
        "records": records if rank == 0 else None,
        "initial": initial,
        "loop_seconds": loop_seconds,
        "steps": spec.steps,
        "timers": timers if timers is not None else Timers(),
        "engine": eng,
    }


def run_serial(setup: RunSetup, ctx: RankContext, timers: Timers | None = None) -> dict:
    """Plain single-rank stepping (strategies.py:335-339): no communication."""
    if ctx.world_size != 1:
        raise ValueError("serial strategy runs on exactly one rank")
    return _run_replicated(setup, None, timers, ctx.device)


def run_particle_decomposition(setup: RunSetup, ctx: RankContext,
                               timers: Timers | None = None) -> dict:
    """Particles split by id, modes replicated, allreduce-only communication
    (strategies.py:342-346)."""
    ctx.space = ctx.world
    return _run_replicated(setup, ctx.world, timers, ctx.device)


def run_domain_decomposition(setup: RunSetup, ctx: RankContext, timers=None) -> dict:
    raise NotImplementedError("domain decomposition (strategies.py:394-434) is outside this "
                              "B200 particle-decomposition build")


def run_parareal(setup: RunSetup, pcfg: PararealConfig, ctx: RankContext, timers=None) -> dict:
    raise NotImplementedError("space-time parareal (strategies.py:507-686) is outside this "
                              "B200 particle-decomposition build")
