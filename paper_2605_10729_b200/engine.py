"""Device-resident particle-decomposition PIF stepper (one rank = one GPU).

This is the B200 replacement of the reference's replicated-mode field operators
and stepping loop (strategies.py:148-173 ``_PifFieldOps``, strategies.py:285-303
``_stepping_loop``).  Per time step, all on one CUDA stream, nothing synchronises
the host:

    interp+push   fused type-2 gather + Boris push + wrap + next cell keys +
                  diagnostic sums               (csrc/particles.cu, 1 launch)
    bin           exclusive scan of cell counts + scatter into the other SoA
                  buffer                         (CUB scan + 1 launch)
    spread        binned register-tiled type-1 spreading   (1 launch)
    modes         cuFFT D2Z + truncate/deconvolve -> allreduce buffer
    allreduce     ONE collective per step of [raw rho_hat | diag(6)]
                  (strategies.py:162-164 and the Recorder's :106 merged)
    fields        finish_deposit + Poisson + energy + Hermitian guard + padded
                  symmetrised half spectra + batched Z2D -> interleaved E grid
    record        3 tiny device copies into the device-side record table

The records come back to the host once, at the end of the run.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _native
from ._device import is_torch, require_cuda
from .diag import DeviceTimers
from .particles import DeviceParticles


class PifEngine:
    """Owns the HBM state of one rank: SoA particles (double buffered), the
    allreduce buffer and the device record table; the plan's native object owns
    the fine grid, spectra, field grid and cell tables."""

    def __init__(self, plan, count: int, device, *, q: float, m: float, externals, dt: float,
                 shape: str = "delta", comm=None, deterministic: bool | None = None):
        torch = require_cuda()
        if shape not in _native.SHAPE:
            raise ValueError(f"unknown shape {shape!r}")
        if dt <= 0:
            raise ValueError(f"dt must be positive, got {dt}")
        self.plan = plan
        self.device = torch.device(device)
        # a native plan holds per-run state (cell tables, field grid, FFT work
        # areas), so every engine owns one; the per-device plan cached on the
        # NufftPlan is reserved for the sequential operator API
        from .nufft import DevicePlan
        idx = self.device.index if self.device.index is not None else torch.cuda.current_device()
        self.dp = DevicePlan(plan, idx)
        self.handle = self.dp.handle
        self.count = int(count)
        self.parts = DeviceParticles(self.count, self.device)
        N3 = plan.N ** 3
        f64 = dict(dtype=torch.float64, device=self.device)
        # allreduce buffer: raw type-1 modes (complex, interleaved) | diag sums | pad
        self.red = torch.zeros(2 * N3 + 8, **f64)
        self.raw = self.red[:2 * N3]
        self.diag = self.red[2 * N3:2 * N3 + 6]
        self.rho = torch.zeros((plan.N,) * 3, dtype=torch.complex128, device=self.device)
        self.scalars = torch.zeros(4, **f64)
        self.configure(q=q, m=m, externals=externals, dt=dt, shape=shape)
        self.comm = comm
        self.rec = None
        self.dtimers = DeviceTimers(enabled=False)
        self.launches = 0   # native kernel launches issued (for bench accounting)
        self.weight_cache = self._enable_weight_cache()
        self.deterministic = False
        if deterministic is None:
            import os
            deterministic = os.environ.get("PIF_DETERMINISTIC", "0").strip() not in (
                "0", "", "false", "off")
        self.set_deterministic(deterministic)

    def set_deterministic(self, on: bool):
        """Bit-reproducible stepping (pif_set_deterministic): stable binning,
        fixed-order plane reduction in the spread, diagnostics from a
        fixed-order pass.  Raises ValueError for windows wider than 8 (the
        DMMA kernels are the only deterministic ones)."""
        _native.call("pif_set_deterministic", self.handle, 1 if on else 0)
        self.deterministic = bool(on)
        if on and self.weight_cache:
            _native.call("pif_set_weight_cache", self.handle, 0)
            self.weight_cache = False

    @property
    def push_aggregated(self) -> bool:
        """Whether the push counts next-cell keys per run (heavy-cell sets;
        decided by the native plan at the first binning after a load)."""
        return bool(_native.load().pif_push_aggregated(self.handle))

    def configure(self, *, q: float, m: float, externals, dt: float, shape: str = "delta"):
        """(Re)set the per-run constants: charge/mass per particle, the Boris
        constants exactly as numpy forms them (pif.py:146-153), the external
        field kind and the particle shape.  Cheap; lets a cached engine serve
        successive pif_step calls."""
        from .pif import boris_constants
        if shape not in _native.SHAPE:
            raise ValueError(f"unknown shape {shape!r}")
        if dt <= 0:
            raise ValueError(f"dt must be positive, got {dt}")
        self.q, self.m, self.dt = float(q), float(m), float(dt)
        half, tq, sq, has_b = boris_constants(self.q / self.m, self.dt, externals.B)
        self.half = float(half)
        self._tq, self._sq = _native.d3(tq), _native.d3(sq)
        self.has_b = int(has_b)
        self.e_kind = _native.EXT[externals.e_kind]
        self.shape = _native.SHAPE[shape]
        self.externals = externals
        return self

    @classmethod
    def cached(cls, plan, count: int, device, *, q: float, m: float, externals, dt: float,
               shape: str = "delta"):
        """The engine a plan keeps for `count` particles on `device`, created on
        first use and reconfigured on every later call (no new cuFFT plans,
        grids or particle store per call).  Used by the reference-shaped
        single-rank API (pif_step, B200FieldOps): not for concurrent use."""
        torch = require_cuda()
        dev = torch.device(device)
        idx = dev.index if dev.index is not None else torch.cuda.current_device()
        key = (idx, int(count))
        with plan._lock:
            cache = plan.__dict__.setdefault("_engines", {})
            eng = cache.get(key)
        if eng is None:
            eng = cls(plan, count, torch.device("cuda", idx), q=q, m=m, externals=externals,
                      dt=dt, shape=shape)
            eng.created_by_cache = True
            with plan._lock:
                cache[key] = eng
            return eng
        eng.created_by_cache = False
        return eng.configure(q=q, m=m, externals=externals, dt=dt, shape=shape)

    def _enable_weight_cache(self) -> bool:
        """Spread -> gather weight reuse (pif_set_weight_cache): the spread of
        step n keeps its 3 x w window weights (192 B per particle at w = 8) and
        the gather of step n+1, which runs at exactly those positions, loads
        them instead of evaluating them again.  On B200 at 2^27 particles this
        trades 2 x 25.8 GB of HBM traffic per step for ~19 clk of FP64 pipe
        work per particle: gather 19.6 -> 17.6 ms, spread 8.8 -> 9.3 ms, step
        -4.8% (profiles/round2/scaling/summary_4xB200.txt); -2.5% at 8 and
        -3.4% at 16 particles per stencil cell, +3% at 1.25, where the gather
        is bound by per-cell work, not weights (profiles/round2/seg_length_ab.txt).
        On by default from 4 particles per stencil cell when HBM has room
        (w <= 8, not in deterministic mode); PIF_WEIGHT_CACHE=0 turns it off,
        =1 asks for it at any density."""
        import os
        torch = require_cuda()
        env = os.environ.get("PIF_WEIGHT_CACHE", "auto").strip().lower()
        want = env not in ("0", "false", "off")
        if env == "auto":
            want = self.count >= 4 * self.plan.n_up ** 3
        on = False
        if want and self.plan.window.w <= 8:
            free, _ = torch.cuda.mem_get_info(self.device)
            on = free > 24 * 8 * self.count + (4 << 30)
        _native.call("pif_set_weight_cache", self.handle, 1 if on else 0)
        return on

    # -- plumbing -------------------------------------------------------------
    def _stream(self):
        return _native.stream_handle(self.device)

    def _soa(self, which="cur"):
        p = self.parts
        i = p.cur if which == "cur" else 1 - p.cur
        return _native.soa_from_store(p.buf[i], p.ids[i], p.count)

    @classmethod
    def for_ensemble(cls, ens, plan, externals, dt, shape="delta", comm=None, device=None,
                     deterministic=None):
        from ._device import default_device
        dev = device if device is not None else default_device(ens.x)
        eng = cls(plan, ens.count, dev, q=ens.q_per_particle, m=ens.m_per_particle,
                  externals=externals, dt=dt, shape=shape, comm=comm,
                  deterministic=deterministic)
        eng.load(ens.x, ens.v, np.arange(ens.count, dtype=np.int64))
        return eng

    def load(self, x, v=None, ids=None):
        """Upload an AoS ensemble and bin it into cell order (v=None: positions
        only, for operators that never push)."""
        torch = require_cuda()
        if not is_torch(x):
            x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
        if v is not None and not is_torch(v):
            v = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64))
        if ids is None:
            ids = torch.arange(self.count, dtype=torch.int64, device=self.device)
        elif not is_torch(ids):
            ids = torch.from_numpy(np.ascontiguousarray(ids, dtype=np.int64))
        self.parts.upload(x.to(self.device), None if v is None else v.to(self.device),
                          ids.to(self.device))
        if self.count:
            s = self._stream()
            cur = self._soa()
            _native.call("pif_wrap_points", self.handle, cur.x, cur.y, cur.z, self.count, s)
            _native.call("pif_bin_keys", self.handle, ctypes.byref(cur),
                         self.parts.key.data_ptr(), self.parts.rank.data_ptr(), s)
            self._bin()

    def load_aos(self, x, v, id0: int):
        """Device (M,3) AoS x, v of ids id0 .. id0+M-1 (host ParticleEnsemble
        layout) -> SoA store, wrapped, binned: one fused pass + perm.
        v=None loads positions only (load_velocities later, before the push)."""
        if self.count:
            cur = self._soa()
            _native.call("pif_load_aos", self.handle, x.data_ptr(),
                         None if v is None else v.data_ptr(), int(id0), ctypes.byref(cur),
                         self.parts.key.data_ptr(), None, self._stream())
            self.launches += 1
            self._bin()

    def load_velocities(self, v):
        """The velocities of a set loaded by load_aos(x, None, id0)."""
        if self.count:
            cur = self._soa()
            _native.call("pif_load_aos_velocities", self.handle, v.data_ptr(), ctypes.byref(cur),
                         self._stream())
            self.launches += 1

    def load_sampled(self, spec, id_range, seed: int | None = None):
        """Generate this rank's slice of the reference ensemble directly into the
        SoA store (no AoS staging: 2^30 particles fit one GPU) and bin it."""
        from .samplers import sample_device_into
        lo, hi = id_range
        if hi - lo != self.count:
            raise ValueError(f"id range {id_range} does not hold {self.count} particles")
        soa = self.parts.soa
        sample_device_into(spec, id_range, [soa[d].data_ptr() for d in range(3)],
                           [soa[3 + d].data_ptr() for d in range(3)], 1, self.device, seed)
        torch = require_cuda()
        ids = self.parts.ids[self.parts.cur]
        torch.arange(lo, hi, dtype=torch.int64, device=self.device, out=ids[:self.count])
        if self.count:
            s = self._stream()
            cur = self._soa()
            _native.call("pif_wrap_points", self.handle, cur.x, cur.y, cur.z, self.count, s)
            _native.call("pif_bin_keys", self.handle, ctypes.byref(cur),
                         self.parts.key.data_ptr(), self.parts.rank.data_ptr(), s)
            self._bin()

    def _bin(self):
        """Cell-ordered view: perm from the keys/ranks of the current buffer."""
        # rank NULL: the in-cell slots come from per-cell cursors in the perm
        # kernel, so the push never waits on a returning atomic
        _native.call("pif_bin_perm", self.handle, self.parts.key.data_ptr(), None, self.count,
                     self.parts.perm.data_ptr(), self._stream())
        # cell scan (CUB: 2 kernels) + perm + work items (segment counts,
        # CUB scan: 2, item table): 7 kernels (profiles/r03_launches.md)
        self.launches += 7

    # -- stages -----------------------------------------------------------------
    def particle_diag(self):
        cur = self._soa()
        _native.call("pif_particle_diag", self.handle, ctypes.byref(cur), self.e_kind,
                     self.diag.data_ptr(), self._stream())
        self.launches += 2

    def spread(self):
        """Binned DMMA spreading into the plan's fine grid (reads through perm)."""
        cur = self._soa()
        _native.call("pif_spread_perm", self.handle, ctypes.byref(cur),
                     self.parts.perm.data_ptr(), None, self.q, self._stream())
        self.launches += 1

    def modes(self):
        """cuFFT D2Z + truncate/deconvolve -> raw modes (head of the allreduce buffer)."""
        _native.call("pif_grid_to_modes", self.handle, self.raw.data_ptr(), self._stream())
        self.launches += 1      # truncate/deconvolve; cuFFT D2Z (library) not counted

    def fft_timing(self, slots: int):
        """Time the next `slots` cuFFT D2Z / Z2D execs with native event pairs
        (pif_fft_timing; 0 disables)."""
        _native.call("pif_fft_timing", self.handle, int(slots))

    def fft_times(self):
        """(mean D2Z ms, mean Z2D ms) over the execs timed since the last call."""
        d, z = ctypes.c_double(), ctypes.c_double()
        nd, nz = ctypes.c_int(), ctypes.c_int()
        _native.call("pif_fft_times", self.handle, ctypes.byref(d), ctypes.byref(z),
                     ctypes.byref(nd), ctypes.byref(nz))
        return (d.value / nd.value if nd.value else None,
                z.value / nz.value if nz.value else None)

    def deposit(self):
        """Scatter stage: spread + modes."""
        self.spread()
        self.modes()

    def allreduce(self):
        if self.comm is not None:
            self.comm.allreduce_sum(self.red, log=not getattr(self, "_capturing", False))

    def solve_fields(self):
        """finish_deposit + Poisson + energy + guard + padded spectra + Z2D."""
        _native.call("pif_solve_fields", self.handle, self.raw.data_ptr(), self.shape,
                     self.rho.data_ptr(), self.scalars.data_ptr(), self._stream())
        self.launches += 5      # poisson, energy, guard (2), pad; cuFFT Z2D (library) not counted

    def interp_push(self):
        """Fused gather + Boris push + next cell keys + diagnostic sums: reads the
        current buffer in cell order (perm), writes the other one, swaps."""
        src, dst = self._soa("cur"), self._soa("alt")
        _native.call("pif_interp_push_perm", self.handle, ctypes.byref(src),
                     self.parts.perm.data_ptr(), ctypes.byref(dst), self.half, self.dt,
                     self._tq, self._sq, self.has_b, self.e_kind, self.parts.key.data_ptr(),
                     None, self.diag.data_ptr(), self._stream())
        self.parts.swap()
        self.launches += 2
        if self.deterministic:      # the fused sums depend on the work-item schedule
            self.particle_diag()

    def set_spread_merge(self, c: int):
        """Merged-column spread for sparse sets: -1 by density (default), 0 off,
        2 or 4 columns per super-column (pif_set_spread_merge)."""
        _native.call("pif_set_spread_merge", self.handle, int(c))

    def spread_merge_used(self) -> int:
        """Columns per super-column of the last spread (1: the column kernel)."""
        return int(_native.load().pif_spread_merge_used(self.handle))

    def split_supported(self) -> bool:
        """pif_interp_split / pif_push_split cover the DMMA kernels (w <= 8)."""
        return bool(_native.load().pif_split_supported(self.handle))

    def gather_split(self, id0: int = 0):
        """Gather half of a split step: E at every particle (positions only;
        the velocities may still be in flight) into a plan-owned (M,3) array,
        row id - id0."""
        cur = self._soa("cur")
        _native.call("pif_interp_split", self.handle, ctypes.byref(cur),
                     self.parts.perm.data_ptr(), int(id0), self._stream())
        self.launches += 1

    def push_rows(self, x, v, r0: int, r1: int):
        """Push half: Boris push of rows [r0, r1) of id-ordered device (M,3)
        x, v in place with the E rows of gather_split; the call reaching row M
        writes the diagnostic sums."""
        _native.call("pif_push_ids", self.handle, x.data_ptr(), v.data_ptr(), self.count,
                     int(r0), int(r1 - r0), self.half, self.dt, self._tq, self._sq, self.has_b,
                     self.e_kind, self.diag.data_ptr(), self._stream())
        self.launches += 1 + (r1 == self.count)

    def rebin(self):
        """Scan the cell counts emitted by interp_push and rebuild perm."""
        if self.count:
            self._bin()

    def gather_push(self):
        self.interp_push()
        self.rebin()

    def record(self, slot: int):
        r = self.rec[slot]
        r[0:1].copy_(self.scalars[0:1])
        r[1:6].copy_(self.diag[0:5])
        r[6:7].copy_(self.scalars[1:2])

    # -- whole runs -----------------------------------------------------------------
    def run(self, steps: int, *, timers=None, graph: bool | None = None):
        """Prime solve + record(0), then `steps` x (gather/push, solve, record)
        (strategies.py:285-303).  Returns the device record table (steps+1, 8):
        [W, sum v.v, sum vx, sum vy, sum vz, sum phi_ext, guard, 0].

        graph=True (default when no timers are requested and steps >= 8):
        the steps are replayed from a CUDA graph of two steps (the particle
        buffers alternate), removing per-launch host overhead; the record slot
        advances through a device-side counter."""
        torch = require_cuda()
        self.rec = torch.zeros((steps + 1, 8), dtype=torch.float64, device=self.device)
        dt = self.dtimers
        dt.enabled = timers is not None
        if graph is None:
            graph = timers is None and steps >= 8 and self._graph_ok()
        self.particle_diag()
        self._solve(dt, record_slot=0)
        self.graph_pairs = 0        # two-step graph replays of the last run
        i = 0
        if graph:
            # two eager steps warm every allocation / plan, then capture
            for _ in range(2):
                self.gather_push()
                self._solve(dt)
                self.record(i + 1)
                i += 1
            pairs = (steps - i) // 2
            if pairs > 0:
                g = self._capture_pair(i + 1)
                for _ in range(pairs):
                    g.replay()
                    self.graph_pairs += 1
                    if self.comm is not None:   # the graph's two collectives
                        self.comm.log_replayed_allreduce(self.red, 2)
                i += 2 * pairs
        for k in range(i, steps):
            with dt.section("Gather"):
                self.gather_push()
            self._solve(dt, record_slot=k + 1)
        if timers is not None:
            dt.flush(timers)
        return self.rec

    def _graph_ok(self) -> bool:
        # NCCL collectives (torchrun ranks or NCCL thread ranks) can be
        # captured; the host-side tree rendezvous of shared-GPU thread ranks cannot
        from .comm import NcclThreadTransport, TorchDistTransport
        return self.comm is None or self.comm.size == 1 or isinstance(
            self.comm.transport, (TorchDistTransport, NcclThreadTransport))

    def _capture_pair(self, first_slot: int):
        """CUDA graph of two full steps recording into rec[slot], rec[slot+1]
        with slot held on the device (advanced by 2 inside the graph)."""
        torch = require_cuda()
        self._slot = torch.tensor([first_slot], dtype=torch.int64, device=self.device)
        self._row = torch.zeros((1, 8), dtype=torch.float64, device=self.device)
        side = torch.cuda.Stream(device=self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        g = torch.cuda.CUDAGraph()
        # capture records the collectives without running them: the call log
        # gets its entries per replay instead (run()); the job's log is shared
        # by all rank threads, so this rank just stops logging while it captures
        self._capturing = True
        try:
            with torch.cuda.stream(side):
                # thread_local: other rank threads keep allocating / launching
                # eagerly while this one captures
                with torch.cuda.graph(g, stream=side, capture_error_mode="thread_local"):
                    for _ in range(2):
                        self.gather_push()
                        self.deposit()
                        self.allreduce()
                        self.solve_fields()
                        self._row[0, 0:1].copy_(self.scalars[0:1])
                        self._row[0, 1:6].copy_(self.diag[0:5])
                        self._row[0, 6:7].copy_(self.scalars[1:2])
                        self.rec.index_copy_(0, self._slot, self._row)
                        self._slot += 1
        finally:
            self._capturing = False
        torch.cuda.current_stream(self.device).wait_stream(side)
        return g

    def _solve(self, dt, record_slot: int | None = None):
        with dt.section("Scatter"):
            self.deposit()
        if self.comm is not None:
            with dt.section("Allreduce"):
                self.allreduce()
        with dt.section("Gather"):
            self.solve_fields()
            if record_slot is not None:   # W and the guard come out of this solve
                self.record(record_slot)

    def step_once(self):
        """One full PD step (used by the bench loop and CUDA-graph capture)."""
        self.gather_push()
        self.deposit()
        self.allreduce()
        self.solve_fields()

    def run_host(self, xh, vh, id0: int, steps: int, energy_out=None, n_chunks: int = 16,
                 trace=None, split=None):
        """pif_step-style stepping of a host-resident ensemble (the reference's
        ParticleEnsemble use, pif.py:178-190): every step uploads x, v ((M,3),
        id order, ids id0 .. id0+M-1) from host memory, bins, deposits, reduces,
        solves, gathers + pushes, scatters back to id order and downloads x, v
        into the same host arrays (energy_out[s] <- the step's field energy).
        split (default True for w <= 8): the gather runs before the velocities
        arrive and only the streaming push waits for them.

        Positions travel first: binning, the deposit, the allreduce and the
        field solve of a step only need x, so they run while v is still being
        uploaded; v is loaded just before the gather + push.  Between steps the
        arrays round-trip chunk by chunk on two copy streams (each chunk's
        upload for step s+1 waits for that chunk's download of step s), x
        chunks first, so both PCIe directions stay busy.  Pin xh / vh (torch
        pin_memory) for asynchronous copies.  trace: a list that receives, per
        step, timing events (step start, x in, fields done, v in, push done,
        downloads done, uploads done) for tools/e2e_timeline.py."""
        torch = require_cuda()
        M, dev = self.count, self.device
        scatter_after = os.environ.get("PIF_E2E_SCATTER", "0") == "1"
        # split (default where the DMMA kernels run): gather E before the
        # velocities arrive, push after; PIF_E2E_SPLIT=0 keeps the fused kernel
        split = (split if split is not None else
                 os.environ.get("PIF_E2E_SPLIT", "1") == "1") and not scatter_after \
            and self.count > 0 and self.split_supported()
        if tuple(xh.shape) != (M, 3) or tuple(vh.shape) != (M, 3):
            raise ValueError(f"host arrays must be ({M}, 3)")
        main = torch.cuda.current_stream(dev)
        down, up = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        if getattr(self, "_stage", None) is None or self._stage[0].shape[0] != M:
            f64 = dict(dtype=torch.float64, device=dev)
            self._stage = (torch.empty((M, 3), **f64), torch.empty((M, 3), **f64))
        xd, vd = self._stage
        step = max(1, -(-M // max(1, n_chunks)))
        bounds = [(i, min(M, i + step)) for i in range(0, M, step)]
        ev = lambda: torch.cuda.Event()  # noqa: E731
        up.wait_stream(main)
        with torch.cuda.stream(up):
            xd.copy_(xh, non_blocking=True)
            x_in = ev()
            x_in.record(up)
            vd.copy_(vh, non_blocking=True)
            v_in = ev()
            v_in.record(up)
        v_evs = [v_in] * len(bounds)   # split: per-chunk velocity arrivals
        # The step's energy leaves by the download stream after that step's
        # x, v chunks: a small D2H on the compute stream would queue on the
        # copy engine behind gigabytes of downloads and stall the next step.
        # It is first copied on the compute stream (an elementwise kernel, not
        # the copy engine) into a per-step device slot.
        ehist = (torch.empty(steps, dtype=torch.float64, device=dev)
                 if energy_out is not None else None)

        def keep_energy(s):
            if ehist is not None:
                torch.mul(self.scalars[0:1], 1.0, out=ehist[s:s + 1])

        def send_energy(s):
            if ehist is not None:
                down.wait_stream(main)
                with torch.cuda.stream(down):
                    energy_out[s:s + 1].copy_(ehist[s:s + 1], non_blocking=True)

        def mark(stream):
            if trace is None:
                return None
            m = torch.cuda.Event(enable_timing=True)
            m.record(stream)
            return m

        for s in range(steps):
            t_start = mark(main)
            main.wait_event(x_in)
            t_x = mark(main)
            self.load_aos(xd, None, id0)
            t_bin = mark(main)
            self._to_cell_order(_native.PIF_PERMUTE_POSITIONS)
            t_perm = mark(main)
            self.deposit()
            t_dep = mark(main)
            self.allreduce()
            self.solve_fields()
            if split:
                # the gather needs positions only: it runs while v is in flight;
                # then each row chunk is pushed as its velocities land and is
                # downloaded as soon as its push ends
                self.gather_split(id0)
                t_fields = mark(main)
                push_ev = []
                for c, (i0, i1) in enumerate(bounds):
                    main.wait_event(v_evs[c])
                    if c == 0:
                        t_v = mark(main)
                    self.push_rows(xd, vd, i0, i1)
                    e = ev()
                    e.record(main)
                    push_ev.append(e)
                keep_energy(s)
                t_push = mark(main)
                last = s == steps - 1
                new_v = []
                for src, dst_h, which in ((xd, xh, "x"), (vd, vh, "v")):
                    for c, (i0, i1) in enumerate(bounds):
                        down.wait_event(push_ev[c])
                        with torch.cuda.stream(down):
                            dst_h[i0:i1].copy_(src[i0:i1], non_blocking=True)
                        if not last:
                            up.wait_stream(down)
                            with torch.cuda.stream(up):
                                src[i0:i1].copy_(dst_h[i0:i1], non_blocking=True)
                            if which == "v":
                                e = ev()
                                e.record(up)
                                new_v.append(e)
                    if not last and which == "x":
                        x_in = ev()
                        x_in.record(up)
                send_energy(s)
                v_evs = new_v
                if trace is not None:
                    trace.append((t_start, t_x, t_fields, t_v, t_push, mark(down), mark(up),
                                  t_bin, t_perm, t_dep))
                continue
            t_fields = mark(main)
            main.wait_event(v_in)
            t_v = mark(main)
            self.load_velocities(vd)
            if scatter_after:
                # push, then one streaming scatter of the pushed set to id order
                self.interp_push()
                self.to_id_order(xd, vd, id0)
                self.rebin()
            else:
                # the push also writes x, v in id order into the staging arrays
                _native.call("pif_set_id_order_output", self.handle, xd.data_ptr(),
                             vd.data_ptr(), int(id0))
                try:
                    self.gather_push()
                finally:
                    _native.call("pif_set_id_order_output", self.handle, None, None, 0)
            keep_energy(s)
            t_push = mark(main)
            down.wait_stream(main)
            last = s == steps - 1
            for src, dst_h, which in ((xd, xh, "x"), (vd, vh, "v")):
                for i0, i1 in bounds:
                    with torch.cuda.stream(down):
                        dst_h[i0:i1].copy_(src[i0:i1], non_blocking=True)
                    if not last:
                        up.wait_stream(down)
                        with torch.cuda.stream(up):
                            src[i0:i1].copy_(dst_h[i0:i1], non_blocking=True)
                if not last:
                    e = ev()
                    e.record(up)
                    if which == "x":
                        x_in = e
                    else:
                        v_in = e
            send_energy(s)
            if trace is not None:
                trace.append((t_start, t_x, t_fields, t_v, t_push, mark(down), mark(up), t_bin,
                              t_perm, t_dep))
        main.wait_stream(down)
        main.wait_stream(up)
        for t in (xd, vd):
            t.record_stream(down)
            t.record_stream(up)

    def _to_cell_order(self, what):
        """Move the current buffer into the cell order of the last binning
        (pif_permute into the other buffer, perm -> identity).  A set loaded
        from id-ordered host arrays is spatially random; read through perm,
        the spread and the gather would gather 8-byte words at random with few
        warps in flight (run_host at 2^27: 74 + 45 ms of compute per step
        instead of ~10 + 28)."""
        if self.count:
            src, dst = self._soa("cur"), self._soa("alt")
            _native.call("pif_permute", self.handle, ctypes.byref(src),
                         self.parts.perm.data_ptr(), ctypes.byref(dst),
                         what | _native.PIF_PERMUTE_RESET, self._stream())
            self.parts.swap()
            self.launches += 1

    def to_id_order(self, x_out=None, v_out=None, id0: int = 0):
        """(M,3) x, v in id order (ids id0 .. id0+M-1) via a device scatter."""
        torch = require_cuda()
        M = self.count
        if x_out is None:
            x_out = torch.empty((M, 3), dtype=torch.float64, device=self.device)
        if v_out is None:
            v_out = torch.empty((M, 3), dtype=torch.float64, device=self.device)
        cur = self._soa()
        _native.call("pif_soa_to_aos", self.handle, ctypes.byref(cur), int(id0), x_out.data_ptr(),
                     v_out.data_ptr(), self._stream())
        return x_out, v_out

    def store_into(self, ens):
        """Copy the particles back into an AoS ensemble, original order."""
        x, v = self.to_id_order()
        if is_torch(ens.x):
            ens.x = x.to(ens.x.device)
            ens.v = v.to(ens.v.device)
        else:
            ens.x = x.cpu().numpy()
            ens.v = v.cpu().numpy()
        return ens

    def rho_field(self):
        from .spectral import FourierField
        f = FourierField(self.plan.N, self.plan.L, self.rho.clone(), "charge-density")
        return f
