"""Host-side logic of the drop-in (CPU only): samplers, plan constants, record
composition, damping fit, output files, timers, and the communicator facade
(thread ranks and a world_size-2 gloo process group)."""

import os

import numpy as np
import pytest

from conftest import golden

import paper_2605_10729_b200 as pb
from paper_2605_10729_b200 import comm, diag, samplers, strategies


SAMP = golden("samplers.npz")


def _sha(*arrays):
    import hashlib
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("key", sorted(SAMP.files))
def test_samplers_bit_identical_to_reference(key):
    _, kind, N, ppm, seed = key.split("_")
    mk = samplers.landau_spec if kind == "landau" else samplers.penning_spec
    spec = mk(N=int(N), ppm=int(ppm), seed=int(seed))
    e = samplers.sample_benchmark(spec, int(seed))
    assert _sha(e.x, e.v, e.ids) == bytes(SAMP[key]).decode()


_M64 = (1 << 64) - 1


def _philox4x64_word(counter, key, j):
    """Pure-Python Philox4x64-10 word j of a stream: the counter / round / key
    schedule the device sampler (csrc/sampler.cu philox_word) implements."""
    c = sum(int(counter[i]) << (64 * i) for i in range(4)) + 1 + (j >> 2)
    c = [(c >> (64 * i)) & _M64 for i in range(4)]
    k0, k1 = int(key[0]), int(key[1])
    for r in range(10):
        if r:
            k0, k1 = (k0 + 0x9E3779B97F4A7C15) & _M64, (k1 + 0xBB67AE8584CAA73B) & _M64
        p0, p1 = 0xD2E7470EE14C6C93 * c[0], 0xCA5A826395121157 * c[2]
        c = [(p1 >> 64) ^ c[1] ^ k0, p1 & _M64, (p0 >> 64) ^ c[3] ^ k1, p0 & _M64]
    return c[j & 3]


@pytest.mark.parametrize("seed,attr", [(0, 0), (0, 5), (7, 2), (123456789, 4)])
def test_device_sampler_stream_layout_matches_numpy(seed, attr):
    """uint64 number j of the reference's (seed, attr) stream is word j & 3 of
    Philox(counter0 + 1 + j // 4, key); uniforms are (raw >> 11) 2^-53."""
    ctr, key = samplers.philox_state(seed, attr)
    gen = np.random.Philox(np.random.SeedSequence((seed, attr)))
    raw = gen.random_raw(23)
    for j in (0, 1, 2, 3, 4, 7, 22):
        assert _philox4x64_word(ctr, key, j) == int(raw[j])
    u = samplers._stream(seed, attr).random(9)
    assert all(u[j] == (int(raw[j]) >> 11) * 2.0 ** -53 for j in range(9))
    # a 256-bit carry across the low counter word
    big = np.array([_M64, 0, 0, 0], dtype=np.uint64)
    gen.state = {"bit_generator": "Philox", "state": {"counter": big, "key": key},
                 "buffer": np.zeros(4, dtype=np.uint64), "buffer_pos": 4, "has_uint32": 0,
                 "uinteger": 0}
    assert _philox4x64_word(big, key, 5) == int(gen.random_raw(6)[5])


def test_id_slices_partition():
    for n_p, size in ((10, 3), (65536, 8), (7, 7), (5, 8)):
        spans = [samplers.id_slice(n_p, r, size) for r in range(size)]
        assert spans[0][0] == 0 and spans[-1][1] == n_p
        assert all(spans[i][1] == spans[i + 1][0] for i in range(size - 1))
        assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def test_plan_constants_match_reference():
    cases = golden("nufft_cases.npz")
    for ci in range(6):
        N, L, eps = cases[f"c{ci}_meta"]
        plan = pb.make_plan(int(N), float(L), float(eps))
        assert np.array_equal(plan.deconv, cases[f"c{ci}_deconv"])
    assert pb.make_plan(16, 1.0, 1e-7).window.w == 8
    assert pb.make_plan(16, 1.0, 1e-16).window.w == 17
    assert pb.make_plan(16, 1.0, 1e-7).n_up == 32


@pytest.mark.parametrize("bad", [dict(N=7, L=1.0, eps=1e-7), dict(N=2, L=1.0, eps=1e-7),
                                 dict(N=8, L=1.0, eps=1e-17), dict(N=8, L=1.0, eps=0.5),
                                 dict(N=8, L=-1.0, eps=1e-7)])
def test_plan_rejects_invalid(bad):
    with pytest.raises(ValueError):
        pb.make_plan(**bad)


def test_damping_fit_matches_reference():
    d = golden("damping.npz")
    got = diag.fit_damping_rate(d["damp_t"], d["damp_w"])
    assert got == pytest.approx(float(d["damp_gamma"][0]), rel=1e-12)


def test_damping_fit_edge_cases():
    t = np.linspace(0, 10, 200)
    assert diag.fit_damping_rate(t, np.full(200, 3.0)) == 0.0
    with pytest.raises(ValueError):
        diag.fit_damping_rate(t, np.linspace(1, 2, 200))


def test_records_compose_like_reference_recorder():
    # table row: [W, sum v.v, sum vx, sum vy, sum vz, sum phi, guard, 0]
    tab = np.array([[2.0, 10.0, 1.0, 2.0, 3.0, 4.0, 0, 0],
                    [1.5, 12.0, 1.0, 2.0, 3.0, 5.0, 0, 0],
                    [1.0, 14.0, 1.0, 2.0, 3.0, 6.0, 0, 0]])
    recs = strategies.records_from_table(tab, steps=2, dt=0.5, q=-2.0, m=3.0, total_charge=-7.0)
    r = recs[2]
    assert r.step == 2 and r.t == 1.0
    assert r.kinetic_energy == 0.5 * 3.0 * 14.0
    assert (r.px, r.py, r.pz) == (3.0, 6.0, 9.0)
    assert r.total_energy == 1.0 + 21.0 + (-2.0 * 6.0)
    assert r.total_charge == -7.0
    every = strategies.records_from_table(tab, steps=2, dt=0.5, q=1, m=1, total_charge=0,
                                          diag_every=2)
    assert [x.step for x in every] == [0, 2]


def test_write_outputs_round_trip(tmp_path):
    recs = [diag.StepRecord(1, 0.1, 1 / 3, 2.0, 3.0, 0.0, 0.0, 0.0, -1.0)]
    t = diag.Timers()
    with t.section("Scatter"):
        pass
    diag.write_outputs(recs, diag.timer_rows([t]), {"a": 1}, str(tmp_path))
    lines = open(tmp_path / "diagnostics.csv").read().splitlines()
    assert lines[0].split(",") == list(diag.CSV_COLUMNS)
    assert lines[1].split(",")[2] == format(1 / 3, ".17g")
    with pytest.raises(FileExistsError):
        diag.write_outputs(recs, [], {}, str(tmp_path))


def test_timers_nest():
    t = diag.Timers()
    with t.section("FinePropagator"):
        with t.section("Scatter"):
            pass
    assert t.inclusive["FinePropagator"] >= t.inclusive["Scatter"]
    assert t.calls["Scatter"] == 1
    with pytest.raises(ValueError):
        with t.section("Nope"):
            pass


# ---------------------------------------------------------------------------
# communicator facade
# ---------------------------------------------------------------------------

def test_thread_allreduce_fixed_tree_order():
    vals = [np.array([1e16, 1.0, -3.0]), np.array([1.0, 2.0, 3.0]), np.array([-1e16, 3.0, 0.5]),
            np.array([1.0, 4.0, 1.5])]
    log = pb.CallLog()
    out = pb.spawn_spmd(4, lambda ctx: ctx.world.allreduce_sum(vals[ctx.world_rank]),
                        call_log=log)
    want = comm.tree_sum(vals)
    for o in out:
        assert np.array_equal(o, want)
    assert log.primitives() == {"allreduce"}
    assert len(log.records) == 4


def test_thread_allreduce_repeated_rounds():
    def prog(ctx):
        acc = []
        for i in range(20):
            acc.append(ctx.world.allreduce_sum(np.array([ctx.world_rank + i], float))[0])
        return acc
    out = pb.spawn_spmd(3, prog)
    assert all(o == [3.0 + 3 * i for i in range(20)] for o in out)


def test_rank_failure_names_rank():
    def prog(ctx):
        if ctx.world_rank == 1:
            raise RuntimeError("boom")
        return ctx.world.allreduce_sum(np.ones(2))
    with pytest.raises(comm.RankFailedError) as ei:
        pb.spawn_spmd(3, prog, watchdog=5.0)
    assert ei.value.rank == 1


def test_allreduce_shape_mismatch():
    def prog(ctx):
        return ctx.world.allreduce_sum(np.ones(2 + ctx.world_rank))
    with pytest.raises(comm.RankFailedError):
        pb.spawn_spmd(2, prog, watchdog=5.0)


def test_deadlock_watchdog():
    def prog(ctx):
        if ctx.world_rank == 0:
            return ctx.world.allreduce_sum(np.ones(1))
        return None
    with pytest.raises(comm.DeadlockError):
        pb.spawn_spmd(2, prog, watchdog=0.5)


def test_spmd_backend_selection(monkeypatch):
    """NCCL thread ranks need one GPU per rank; without GPUs (this host) the
    fixed-order tree rendezvous serves spawn_spmd, and PIF_SPMD_BACKEND or the
    backend argument pick explicitly."""
    monkeypatch.delenv("PIF_SPMD_BACKEND", raising=False)
    assert comm._default_backend(1) == "threads"
    assert comm._default_backend(4) in ("threads", "nccl")
    monkeypatch.setenv("PIF_SPMD_BACKEND", "threads")
    assert comm._default_backend(8) == "threads"
    seen = pb.spawn_spmd(2, lambda ctx: type(ctx.world.transport).__name__, backend="threads")
    assert seen == ["ThreadTransport", "ThreadTransport"]
    with pytest.raises(ValueError):
        pb.spawn_spmd(2, lambda ctx: None, backend="mpi")


def test_p2p_is_outside_this_build():
    with pytest.raises(comm.CommError):
        pb.spawn_spmd(1, lambda ctx: ctx.world.send(0, 1))


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    log = comm.CallLog()
    ctx = comm.context_from_env(call_log=log, backend="gloo")
    a = ctx.world.allreduce_sum(np.array([rank + 1.0, 2.0 * rank]))
    t = torch.tensor([1.0, rank + 0.5], dtype=torch.float64)
    ctx.world.allreduce_sum(t)
    q.put((rank, a.tolist(), t.tolist(), sorted(log.primitives())))
    dist.destroy_process_group()


def test_torch_dist_gloo_world_size_2():
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    for rank, a, t, prims in res:
        assert a == [3.0, 2.0]
        assert t == [2.0, 2.0]
        assert prims == ["allreduce"]


def test_out_of_scope_strategies_raise():
    with pytest.raises(NotImplementedError):
        pb.run_domain_decomposition(None, None)
    with pytest.raises(NotImplementedError):
        pb.pic_step()


def test_criterion_9_parameter_fidelity():
    """test_acceptance.py:294-310: the benchmark specs' defaults."""
    import numpy as np
    lan = samplers.landau_spec()
    assert lan.L == 4 * np.pi and lan.Q_e == -lan.L ** 3
    assert (lan.k, lan.alpha, lan.dt, lan.steps) == (0.5, 0.05, 0.003125, 768)
    pen = samplers.penning_spec()
    assert (pen.L, pen.Q_e) == (25.0, -1562.5)
    assert pen.B_ext == (0.0, 0.0, 5.0) and pen.stds == (2.0, 1.0, 3.0)
    assert pen.e_kind == "quadrupole"
