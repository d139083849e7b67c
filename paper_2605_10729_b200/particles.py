"""Macro-particle ensembles: the reference's AoS container plus the HBM store.

``ParticleEnsemble`` keeps the reference's public shape (particles.py:10-62):
(count, 3) positions/velocities, int64 ids, uniform q and m, global totals.  Its
arrays may be numpy (host) or torch CUDA tensors (device); the operator API
returns the same kind it is given.

``DeviceParticles`` is the B200 layout the hot path runs on: structure of
arrays (x, y, z, vx, vy, vz as separate fp64 vectors, ids int64), double
buffered so binning can scatter from one copy into the other, resident in HBM
for the whole run (48 B + 8 B per particle per buffer).
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


@dataclass
class ParticleEnsemble:
    x: object                # (count, 3) positions in [0, L)
    v: object                # (count, 3) velocities
    ids: object              # (count,) int64
    q_per_particle: float
    m_per_particle: float
    total_charge: float
    total_mass: float
    global_count: int

    def __post_init__(self):
        if _is_torch(self.x):
            import torch
            self.x = self.x.to(torch.float64).contiguous()
            self.v = self.v.to(device=self.x.device, dtype=torch.float64).contiguous()
            self.ids = self.ids.to(device=self.x.device, dtype=torch.int64).contiguous()
        else:
            self.x = np.ascontiguousarray(self.x, dtype=np.float64)
            self.v = np.ascontiguousarray(self.v, dtype=np.float64)
            self.ids = np.ascontiguousarray(self.ids, dtype=np.int64)
        n = self.x.shape[0]
        if tuple(self.x.shape) != (n, 3) or tuple(self.v.shape) != (n, 3) \
                or tuple(self.ids.shape) != (n,):
            raise ValueError(f"inconsistent particle batch: x{tuple(self.x.shape)} "
                             f"v{tuple(self.v.shape)} ids{tuple(self.ids.shape)}")

    @property
    def count(self) -> int:
        return int(self.x.shape[0])

    def copy(self) -> "ParticleEnsemble":
        return replace(self, x=self.x.copy() if not _is_torch(self.x) else self.x.clone(),
                       v=self.v.copy() if not _is_torch(self.v) else self.v.clone(),
                       ids=self.ids.copy() if not _is_torch(self.ids) else self.ids.clone())

    def take(self, index) -> "ParticleEnsemble":
        return replace(self, x=self.x[index], v=self.v[index], ids=self.ids[index])

    def sort_by_id(self) -> "ParticleEnsemble":
        if _is_torch(self.ids):
            import torch
            return self.take(torch.argsort(self.ids, stable=True))
        return self.take(np.argsort(self.ids, kind="stable"))

    @staticmethod
    def concat(parts: list["ParticleEnsemble"]) -> "ParticleEnsemble":
        if not parts:
            raise ValueError("concat of zero parts")
        head = parts[0]
        if _is_torch(head.x):
            import torch
            cat = torch.cat
        else:
            cat = np.concatenate
        return replace(head, x=cat([p.x for p in parts], 0), v=cat([p.v for p in parts], 0),
                       ids=cat([p.ids for p in parts]))


def wrap_positions(x, L: float):
    """x mod L in [0, L), guarding the round-up-to-L edge (particles.py:65-70)."""
    if _is_torch(x):
        import torch
        w = torch.remainder(x, L)
        return torch.where(w >= L, w - L, w)
    w = np.mod(x, L)
    w[w >= L] -= L
    return w


def minimum_image(delta, L: float):
    """Shortest periodic representative (particles.py:73-75)."""
    if _is_torch(delta):
        import torch
        return delta - L * torch.round(delta / L)
    return delta - L * np.round(delta / L)


class DeviceParticles:
    """Double-buffered SoA particle store in HBM (one per rank/GPU).

    Buffer ``cur`` holds the particles; ``perm`` lists them in ES-stencil cell
    order (binning never moves particle data).  The gather+push kernel reads
    ``cur`` through ``perm`` and writes the updated particles, in that order,
    to the other buffer, which becomes ``cur``; it also emits their next cell
    keys, from which binning rebuilds ``perm``.
    """

    FIELDS = ("x", "y", "z", "vx", "vy", "vz")

    def __init__(self, count: int, device, capacity: int | None = None):
        import torch
        self.count = int(count)
        cap = max(1, int(capacity if capacity is not None else count))
        self.device = torch.device(device)
        f64 = dict(dtype=torch.float64, device=self.device)
        self.buf = [torch.empty((6, cap), **f64), torch.empty((6, cap), **f64)]
        self.ids = [torch.empty(cap, dtype=torch.int64, device=self.device),
                    torch.empty(cap, dtype=torch.int64, device=self.device)]
        self.key = torch.empty(cap, dtype=torch.int32, device=self.device)
        self.rank = torch.empty(cap, dtype=torch.int32, device=self.device)
        self.perm = torch.empty(cap, dtype=torch.int32, device=self.device)
        self.cur = 0

    @property
    def soa(self):
        return self.buf[self.cur]

    @property
    def alt(self):
        return self.buf[1 - self.cur]

    def swap(self):
        self.cur = 1 - self.cur

    def upload(self, x, v, ids):
        """Copy AoS (M,3) x, v and (M,) ids (numpy or torch) into buffer cur."""
        import torch
        M = self.count
        xt = torch.as_tensor(x, dtype=torch.float64).reshape(M, 3)
        soa = self.buf[self.cur]
        soa[0:3, :M].copy_(xt.t(), non_blocking=True)
        if v is None:
            soa[3:6, :M].zero_()
        else:
            vt = torch.as_tensor(v, dtype=torch.float64).reshape(M, 3)
            soa[3:6, :M].copy_(vt.t(), non_blocking=True)
        self.ids[self.cur][:M].copy_(torch.as_tensor(ids, dtype=torch.int64), non_blocking=True)

    def download(self, sort_by_id: bool = True):
        """Return AoS (x, v, ids) torch tensors on the device (id order if asked)."""
        import torch
        M = self.count
        soa = self.buf[self.cur][:, :M]
        ids = self.ids[self.cur][:M]
        x = soa[0:3].t().contiguous()
        v = soa[3:6].t().contiguous()
        if sort_by_id:
            order = torch.argsort(ids, stable=True)
            return x[order], v[order], ids[order]
        return x, v, ids
