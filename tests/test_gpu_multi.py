"""Particle decomposition across processes over NCCL (one rank per GPU), the
torchrun layout bench.py uses.  Needs >= 2 GPUs; skipped otherwise."""

import os
import socket

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import paper_2605_10729_b200 as pb
    from paper_2605_10729_b200 import comm
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    log = comm.CallLog()
    ctx = comm.context_from_env(call_log=log, backend="nccl")
    spec = pb.landau_spec(N=16, ppm=16, dt=0.05, steps=20, seed=0)
    res = pb.run_particle_decomposition(pb.RunSetup(spec=spec, eps=1e-7), ctx)
    tr = None
    if rank == 0:
        tr = [[r.field_energy, r.kinetic_energy, r.total_energy]
              for r in [res["initial"]] + res["records"]]
    q.put((rank, tr, sorted(log.primitives()), len(log.records)))
    dist.barrier()
    dist.destroy_process_group()
    del torch


def test_nccl_pd_two_processes_matches_reference(cuda):
    torch = cuda
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=300) for _ in range(2)), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
    ref = golden("config1.npz")["landau_pd2_trace"][:, 2:5]
    got = np.array(out[0][1])
    assert np.max(np.abs(got - ref) / np.abs(ref)) <= 1e-10
    for rank, _, prims, n in out:
        assert prims == ["allreduce"]
        assert n == 21          # one collective per step (+ the priming solve)


def test_cli_under_torchrun_two_gpus(cuda, tmp_path):
    """`torchrun -m paper_2605_10729_b200.cli --strategy pd` — one process per GPU."""
    torch = cuda
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import subprocess
    import sys
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = tmp_path / "run"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           "-m", "paper_2605_10729_b200.cli", "--benchmark", "landau", "--strategy", "pd",
           "--modes", "16", "--ppm", "16", "--dt", "0.05", "--steps", "20",
           "--ranks-space", "2", "--out-dir", str(out), "--log-comm"]
    proc = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, proc.stderr[-3000:]
    assert "final_field_energy=" in proc.stdout
    import csv
    with open(out / "diagnostics.csv") as f:
        rows = list(csv.DictReader(f))
    ref = golden("config1.npz")["landau_pd2_trace"][1:, 2]
    got = np.array([float(r["field_energy"]) for r in rows])
    assert np.max(np.abs(got - ref) / np.abs(ref)) <= 1e-10
    with open(out / "timers.csv") as f:
        assert {r["rank"] for r in csv.DictReader(f)} == {"0", "1"}


# ---------------------------------------------------------------------------
# the reference's in-process model: spawn_spmd thread ranks over NCCL
# (comm.py:483-528; communicators from one ncclCommInitAll, pif_comm_init_all)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("P", [2, 4])
def test_spawn_spmd_thread_ranks_run_pd_over_nccl_with_graphs(P, cuda):
    torch = cuda
    if torch.cuda.device_count() < P:
        pytest.skip(f"needs {P} GPUs")
    import paper_2605_10729_b200 as pb
    from paper_2605_10729_b200 import comm
    spec = pb.landau_spec(N=16, ppm=16, dt=0.05, steps=20, seed=0)
    setup = pb.RunSetup(spec=spec, eps=1e-7)
    log = comm.CallLog()
    seen = []

    def program(ctx):
        seen.append(type(ctx.world.transport).__name__)
        return pb.run_particle_decomposition(setup, ctx)

    res = pb.spawn_spmd(P, program, call_log=log)
    assert set(seen) == {"NcclThreadTransport"}
    for rank, r in enumerate(res):
        assert r["engine"].graph_pairs > 0              # steps replayed from CUDA graphs
        assert r["engine"].device.index == rank
    cfg = golden("config1.npz")
    got = np.array([[r.field_energy, r.kinetic_energy, r.total_energy]
                    for r in [res[0]["initial"]] + res[0]["records"]])
    ref = cfg["landau_pd2_trace" if P == 2 else "landau_trace"][:, 2:5]
    assert np.max(np.abs(got - ref) / np.abs(ref)) <= 1e-10
    assert log.primitives() == {"allreduce"}
    assert len(log.records) == P * (spec.steps + 1)     # one collective per step and rank


def test_nccl_thread_transport_reduces_numpy_and_tensors(cuda):
    torch = cuda
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import paper_2605_10729_b200 as pb

    def program(ctx):
        r = ctx.world_rank
        a = ctx.world.allreduce_sum(np.array([1.0 + r, 2.0 * r, 1j * r]))
        t = torch.full((5,), float(r + 1), dtype=torch.float64, device=ctx.device)
        ctx.world.allreduce_sum(t)
        return a, t.cpu().numpy()

    out = pb.spawn_spmd(2, program, backend="nccl")
    for a, t in out:
        assert np.array_equal(a, np.array([3.0, 2.0, 1j]))
        assert np.array_equal(t, np.full(5, 3.0))
