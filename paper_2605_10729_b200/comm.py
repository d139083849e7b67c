"""Communicator facade: the reference's SPMD surface over two transports.

The reference (/root/reference/pkg/src/pifsim/comm.py) runs ranks as threads in
one process with a deterministic tree allreduce.  The particle-decomposition
path only needs ``allreduce_sum`` (strategies.py:124-128, 162-164), so this
module keeps the same facade — ``Comm`` (rank, size, label, allreduce_sum),
``CallLog``, ``RankContext``, ``spawn_spmd``, the error types — over:

* ``NcclThreadTransport``: ranks are threads of this process (spawn_spmd),
  each driving its own GPU; the allreduce is one in-place ``ncclAllReduce``
  per call on the rank's stream, over communicators made by one
  ``ncclCommInitAll`` (libpifb200 ``pif_comm_init_all`` / ``pif_allreduce_f64``),
  so CUDA graphs can capture it.  The default whenever every rank has a GPU of
  its own.
* ``ThreadTransport``: the same thread ranks when GPUs are shared (or none):
  a rendezvous whose last arrival reduces in fixed binary-tree order
  (comm.py:329-339 semantics) over numpy arrays or CUDA tensors.
* ``TorchDistTransport``: one process per GPU (torchrun), the allreduce is one
  in-place NCCL ``all_reduce`` over NVLink/NVSwitch (gloo for CPU tests).

Point-to-point, alltoall and split (domain decomposition / parareal) are out of
scope for this tier and raise.
"""

from __future__ import annotations

import csv
import os
import threading
import time
from dataclasses import dataclass
from typing import Any, Callable

import numpy as np


class CommError(RuntimeError):
    pass


class DeadlockError(CommError):
    """A blocking collective exceeded the watchdog timeout."""


class RankFailedError(CommError):
    def __init__(self, rank: int, message: str):
        super().__init__(message)
        self.rank = rank


class _JobAborted(CommError):
    pass


@dataclass
class CallRecord:
    rank: int
    primitive: str
    comm: str
    peer: int
    nbytes: int


class CallLog:
    """Thread-safe record of every data-moving primitive (comm.py:195-223)."""

    def __init__(self):
        self._lock = threading.Lock()
        self.records: list[CallRecord] = []

    def add(self, rank, primitive, comm, peer, nbytes):
        with self._lock:
            self.records.append(CallRecord(rank, primitive, comm, peer, int(nbytes)))

    def primitives(self) -> set[str]:
        return {r.primitive for r in self.records}

    def write_csv(self, path) -> None:
        with open(path, "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["rank", "primitive", "comm", "peer", "nbytes"])
            for r in self.records:
                w.writerow([r.rank, r.primitive, r.comm, r.peer, r.nbytes])


def _nbytes(a) -> int:
    if type(a).__module__.startswith("torch"):
        return a.numel() * a.element_size()
    return np.asarray(a).nbytes


def tree_sum(arrays: list):
    """Fixed binary-tree reduction order (bit-reproducible for a given layout)."""
    level = list(arrays)
    while len(level) > 1:
        nxt = [level[i] + level[i + 1] for i in range(0, len(level) - 1, 2)]
        if len(level) % 2:
            nxt.append(level[-1])
        level = nxt
    return level[0]


# ---------------------------------------------------------------------------
# in-process thread transport
# ---------------------------------------------------------------------------

class _Job:
    def __init__(self, watchdog: float, call_log: CallLog | None):
        self.watchdog = watchdog
        self.call_log = call_log
        self.failed = threading.Event()
        self.failures: list[tuple[int, BaseException]] = []
        self._lock = threading.Lock()

    def fail(self, rank, exc):
        with self._lock:
            self.failures.append((rank, exc))
        self.failed.set()

    def log(self, *rec):
        if self.call_log is not None:
            self.call_log.add(*rec)


class ThreadTransport:
    """Rendezvous of `size` rank threads; the last arrival reduces."""

    def __init__(self, job: _Job, size: int, label: str):
        self.job, self.size, self.label = job, size, label
        self._cv = threading.Condition()
        self._gen = 0
        self._slots: dict[int, Any] = {}
        self._result: Any = None
        self._readers = 0

    def allreduce(self, rank: int, value):
        deadline = time.monotonic() + self.job.watchdog
        with self._cv:
            while self._readers:          # previous round still being read
                self._wait(rank, deadline)
            gen = self._gen
            self._slots[rank] = value
            if len(self._slots) == self.size:
                ordered = [self._slots[r] for r in range(self.size)]
                shapes = {tuple(a.shape) for a in ordered}
                if len(shapes) != 1:
                    self._result = CommError(
                        f"allreduce length mismatch on '{self.label}': {sorted(shapes)}")
                else:
                    self._result = _reduce_any(ordered)
                self._slots = {}
                self._readers = self.size
                self._gen += 1
                self._cv.notify_all()
            while self._gen == gen:
                self._wait(rank, deadline)
            res = self._result
            self._readers -= 1
            if self._readers == 0:
                self._cv.notify_all()
        if isinstance(res, Exception):
            raise res
        return res

    def _wait(self, rank, deadline):
        self._cv.wait(timeout=0.02)
        if self.job.failed.is_set():
            raise _JobAborted("aborted: another rank failed")
        if time.monotonic() > deadline:
            raise DeadlockError(f"rank {rank} blocked in allreduce on comm '{self.label}'")


def _reduce_any(ordered):
    first = ordered[0]
    if type(first).__module__.startswith("torch"):
        dev = first.device
        return tree_sum([a.to(dev) for a in ordered])
    return tree_sum([np.asarray(a) for a in ordered])


class NcclThreadTransport:
    """Thread ranks with one GPU each; allreduce = ncclAllReduce (in place, on
    the calling thread's current stream).  numpy values go through a device
    copy of the rank's GPU."""

    def __init__(self, job: _Job, size: int, devices: list, label: str = "world"):
        import ctypes

        from . import _native
        self.job, self.size, self.label = job, size, label
        self.devices = [int(d) for d in devices]
        lib = _native.load()
        arr = (ctypes.c_int * size)(*self.devices)
        out = (ctypes.c_void_p * size)()
        _native.check(lib.pif_comm_init_all(size, arr, out), "pif_comm_init_all")
        self._comms = list(out)
        self._lib = lib

    def allreduce(self, rank: int, value):
        import torch

        from . import _native
        dev = torch.device("cuda", self.devices[rank])
        if type(value).__module__.startswith("torch"):
            t = value
            if t.device != dev or t.dtype != torch.float64 or not t.is_contiguous():
                raise CommError(f"rank {rank}: NCCL allreduce needs a contiguous float64 "
                                f"tensor on {dev}, got {t.dtype} on {t.device}")
            _native.check(self._lib.pif_allreduce_f64(self._comms[rank], t.data_ptr(), t.numel(),
                                                      _native.stream_handle(dev)),
                          "pif_allreduce_f64")
            return t
        arr = np.asarray(value)
        cplx = np.iscomplexobj(arr)
        flat = np.ascontiguousarray(arr, dtype=np.complex128 if cplx else np.float64)
        t = torch.from_numpy(flat.view(np.float64).reshape(-1).copy()).to(dev)
        _native.check(self._lib.pif_allreduce_f64(self._comms[rank], t.data_ptr(), t.numel(),
                                                  _native.stream_handle(dev)), "pif_allreduce_f64")
        out = t.cpu().numpy()
        return (out.view(np.complex128) if cplx else out).reshape(arr.shape)

    def close(self):
        for c in self._comms:
            if c:
                self._lib.pif_comm_destroy(c)
        self._comms = [None] * self.size


# ---------------------------------------------------------------------------
# torch.distributed transport (NCCL on GPUs, gloo on CPU)
# ---------------------------------------------------------------------------

class TorchDistTransport:
    def __init__(self, group=None, label: str = "world"):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.size = dist.get_world_size(group)
        self.label = label
        self.job = _Job(watchdog=float("inf"), call_log=None)

    def allreduce(self, rank: int, value):
        import torch
        dist = self.dist
        if type(value).__module__.startswith("torch"):
            dist.all_reduce(value, op=dist.ReduceOp.SUM, group=self.group)
            return value
        backend = dist.get_backend(self.group)
        dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else "cpu"
        t = torch.as_tensor(np.asarray(value), device=dev).clone()
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t.cpu().numpy()


class Comm:
    """Rank-local view of one communicator (comm.py:346-408 surface)."""

    def __init__(self, transport, rank: int):
        self._t = transport
        self.rank = rank

    @property
    def size(self) -> int:
        return self._t.size

    @property
    def label(self) -> str:
        return self._t.label

    @property
    def transport(self):
        return self._t

    def allreduce_sum(self, values, log: bool = True):
        """Element-wise sum over ranks.  numpy in -> new numpy out (reference
        semantics); torch tensor in -> reduced in place and returned.
        log=False: not recorded in the CallLog (a CUDA-graph capture, whose
        replays are logged instead)."""
        if log:
            self._t.job.log(self.rank, "allreduce", self.label, -1, _nbytes(values))
        if self.size == 1:
            if type(values).__module__.startswith("torch"):
                return values
            return np.array(values, copy=True)
        res = self._t.allreduce(self.rank, values)
        if type(values).__module__.startswith("torch"):
            if res is not values:
                values.copy_(res)
            return values
        return np.array(res, copy=True)

    def log_replayed_allreduce(self, values, times: int = 1):
        """Record allreduces a CUDA-graph replay issued without passing through
        allreduce_sum (the graph captured them once), so the CallLog keeps one
        entry per executed collective."""
        for _ in range(times):
            self._t.job.log(self.rank, "allreduce", self.label, -1, _nbytes(values))

    def send(self, dest, payload):
        raise CommError("point-to-point send is outside the particle-decomposition path")

    def recv(self, src):
        raise CommError("point-to-point recv is outside the particle-decomposition path")

    def alltoall(self, blocks):
        raise CommError("alltoall is outside the particle-decomposition path")

    def split(self, color, key, label=None):
        raise CommError("communicator split is outside the particle-decomposition path")


@dataclass
class RankContext:
    world: Comm
    space: Comm | None = None
    time: Comm | None = None
    slab: Any = None
    device: Any = None        # CUDA device this rank drives

    @property
    def world_rank(self) -> int:
        return self.world.rank

    @property
    def world_size(self) -> int:
        return self.world.size


def _rank_device(rank: int):
    try:
        import torch
        if torch.cuda.is_available():
            return torch.device("cuda", rank % torch.cuda.device_count())
    except Exception:  # noqa: BLE001
        pass
    return None


def _default_backend(num_ranks: int) -> str:
    """"nccl" when every rank thread gets a GPU of its own, else "threads"
    (env PIF_SPMD_BACKEND overrides)."""
    want = os.environ.get("PIF_SPMD_BACKEND", "").strip().lower()
    if want in ("nccl", "threads"):
        return want
    try:
        import torch
        if num_ranks > 1 and torch.cuda.is_available() and \
                num_ranks <= torch.cuda.device_count():
            return "nccl"
    except Exception:  # noqa: BLE001
        pass
    return "threads"


def spawn_spmd(num_ranks: int, program: Callable[[RankContext], Any], *,
               watchdog: float = 60.0, call_log: CallLog | None = None,
               backend: str | None = None) -> list:
    """Run `program` on `num_ranks` in-process rank threads (comm.py:483-528
    contract: results in rank order, any failure aborts the job and names the
    rank).  Rank r drives CUDA device r mod device_count.  backend "nccl"
    (default when each rank has its own GPU) reduces with ncclAllReduce over
    communicators from one ncclCommInitAll; "threads" with the fixed-order
    tree rendezvous."""
    if num_ranks < 1:
        raise ValueError(f"num_ranks must be >= 1, got {num_ranks}")
    backend = backend or _default_backend(num_ranks)
    if backend not in ("nccl", "threads"):
        raise ValueError(f"unknown spmd backend {backend!r}")
    job = _Job(watchdog, call_log)
    if backend == "nccl" and num_ranks > 1:
        transport = NcclThreadTransport(job, num_ranks, list(range(num_ranks)), "world")
    else:
        transport = ThreadTransport(job, num_ranks, "world")
    results: list = [None] * num_ranks

    def worker(rank):
        try:
            dev = _rank_device(rank)
            if dev is not None:
                import torch
                torch.cuda.set_device(dev)
            results[rank] = program(RankContext(world=Comm(transport, rank), device=dev))
        except _JobAborted:
            pass
        except BaseException as exc:  # noqa: BLE001
            job.fail(rank, exc)

    threads = [threading.Thread(target=worker, args=(r,), name=f"spmd-rank-{r}", daemon=True)
               for r in range(num_ranks)]
    for t in threads:
        t.start()
    # a rank that died leaves its peers waiting inside a collective (NCCL
    # kernels never time out): give them `watchdog` seconds, then report
    failed_at = None
    while any(t.is_alive() for t in threads):
        for t in threads:
            t.join(timeout=0.05)
        if job.failed.is_set():
            failed_at = failed_at or time.monotonic()
            if time.monotonic() - failed_at > watchdog:
                break
    hung = [t for t in threads if t.is_alive()]
    if not hung and isinstance(transport, NcclThreadTransport):
        transport.close()
    if job.failures:
        dead = [(r, e) for r, e in job.failures if isinstance(e, DeadlockError)]
        other = [(r, e) for r, e in job.failures if not isinstance(e, DeadlockError)]
        if other:
            rank, exc = other[0]
            raise RankFailedError(rank, f"rank {rank} failed: {exc!r}") from exc
        rank, exc = dead[0]
        raise DeadlockError(f"deadlock: blocked ranks {sorted(r for r, _ in dead)}; "
                            f"first: {exc}") from exc
    return results


def context_from_env(call_log: CallLog | None = None, backend: str | None = None) -> RankContext:
    """RankContext for a torchrun-launched process (one rank per GPU, NCCL)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)
    t = TorchDistTransport()
    t.job.call_log = call_log
    rank = dist.get_rank()
    dev = None
    if torch.cuda.is_available():
        local = int(os.environ.get("LOCAL_RANK", rank % torch.cuda.device_count()))
        dev = torch.device("cuda", local)
        torch.cuda.set_device(dev)
    return RankContext(world=Comm(t, rank), device=dev)
