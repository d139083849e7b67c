#!/usr/bin/env python
"""bench.py — particle-decomposition PIF time step on B200 (one JSON line).

Default workload (BASELINE.json configs[1], the metric's config): 3D-3V Landau
damping, 64^3 modes, 2^27 particles per GPU (ppm 512), eps 1e-7 (w = 8),
dt 0.003125, fp64.  A "step" is one full PD-PIF step: fused gather+push,
binning, spreading, D2Z + truncate, ONE allreduce of [rho_hat | diag] (N > 1),
field solve + 3x Z2D.  N GPUs run as torchrun ranks over NCCL; per-GPU work is
fixed (weak scaling: N = 8 is the north-star 2^30-particle run) unless
--scaling strong.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

--impl reference times the reference algorithm's CPU implementation (the C +
numpy oracle port in oracle/, all host cores) on a bounded sample of the same
workload; under torchrun only rank 0 runs it.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle-steps/sec (Landau 3D-3V, 64^3 modes) at 1/2/4/8 B200; % roofline"
UNIT = "particle-steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--kind", default="landau", choices=["landau", "penning"])
    ap.add_argument("--N", type=int, default=64)
    ap.add_argument("--ppm", type=int, default=512, help="particles per mode (per GPU if weak)")
    ap.add_argument("--eps", type=float, default=1e-7)
    ap.add_argument("--dt", type=float, default=0.003125)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--cpu-particles", type=int, default=1 << 24,
                    help="particles in the CPU (reference-algorithm) sample")
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--cpu-max-steps", type=int, default=8,
                    help="cap on the reference arm's timed steps (bounded run time)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None,
                    help="host-streamed steps in the e2e measurement (default min(--steps, 10))")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def workload_config(a, world):
    from paper_2605_10729_b200.nufft import make_plan
    w = make_plan(a.N, 1.0, a.eps).window.w
    per_gpu = a.ppm * a.N ** 3 if a.scaling == "weak" else (a.ppm * a.N ** 3) // world
    glob = per_gpu * world if a.scaling == "weak" else a.ppm * a.N ** 3
    name = "Landau damping" if a.kind == "landau" else "Penning trap"
    return {
        "workload": f"3D-3V {name}, {a.N}^3 modes, {glob} particles "
                    f"({per_gpu}/GPU), eps {a.eps:g} (w={w}), dt {a.dt:g}, fp64, "
                    f"particle decomposition",
        "modes_per_dim": a.N, "fine_grid": 2 * a.N, "window_w": w, "eps": a.eps, "dt": a.dt,
        "particles_per_gpu": per_gpu, "global_particles": glob, "parallelism": f"pd{world}",
        "l2": "particle SoA (48 B/particle) >> 126 MB L2: inputs larger than L2, no flush",
    }, w, per_gpu, glob


# ---------------------------------------------------------------------------
# clocks sampling (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.index)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline / reference arm (oracle port of the reference algorithm)
# ---------------------------------------------------------------------------

def cpu_reference_run(a, particles: int, steps: int, warmup: int, full_particles: int):
    """Oracle PD on all host cores (one rank thread per core, like the
    reference's spawn_spmd PD run).  Returns a dict: measured particle-steps/s
    at `particles`, the per-step phase split, and the explicit extrapolation to
    `full_particles` (particle phases scale with the count, the mode-space
    FFT phases do not)."""
    import numpy as np  # noqa: F401
    from oracle import pif_oracle as o
    from paper_2605_10729_b200.samplers import landau_spec, penning_spec, sample_benchmark
    cores = os.cpu_count() or 1
    ppm = max(1, particles // a.N ** 3)
    mk = landau_spec if a.kind == "landau" else penning_spec
    spec = mk(N=a.N, ppm=ppm, dt=a.dt, seed=0)
    ens = sample_benchmark(spec, 0)
    plan = o.make_plan(a.N, spec.L, a.eps)
    run = o.PDRun(plan, ens.x, ens.v, ens.q_per_particle, ens.m_per_particle, L=spec.L,
                  B=spec.B_ext, e_kind=spec.e_kind, dt=a.dt, ranks=cores)
    for _ in range(warmup):
        run.step()
    run.phase_s = dict.fromkeys(run.PHASES, 0.0)
    t0 = time.perf_counter()
    for _ in range(steps):
        run.step()
    sec = (time.perf_counter() - t0) / steps
    M = ens.count
    split = {k: v / steps for k, v in run.phase_s.items()}
    linear = split["spread"] + split["interp"] + split["push"]
    fixed = split["fftn"] + split["field_grids"]
    other = max(0.0, sec - linear - fixed)          # Poisson, energy, tree sum (fixed)
    scale = full_particles / M
    t_full = linear * scale + fixed + other
    sample = (f"{M} particles ({ppm}/mode) of the same {a.N}^3 workload (eps {a.eps:g}), "
              f"{steps} PD steps on {cores} host threads (oracle port of the reference "
              "algorithm: C window kernels + numpy pocketfft; one rank slice per thread)")
    return {
        "value": M / sec, "cores": cores, "sample": sample, "sec_per_step": sec,
        "particles_timed": M, "steps_timed": steps,
        "split_s_per_step": {**{k: round(v, 6) for k, v in split.items()},
                             "other": round(other, 6)},
        "extrapolated": {"particles": full_particles, "value": full_particles / t_full,
                         "sec_per_step": t_full,
                         "how": "particle phases (spread, interp, push) x particles ratio + "
                                "fixed mode-space phases (fftn, 3x ifftn, Poisson, sums)"},
    }


def run_reference(a):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg, w, per_gpu, glob = workload_config(a, world)
    # K timed steps after W warm-ups, each one PD step over a bounded sample
    # (cpu_particles) of the workload; capped so the arm ends within minutes
    steps = max(1, min(a.steps, a.cpu_max_steps))
    warm = max(0, min(a.warmup, 1))
    r = cpu_reference_run(a, a.cpu_particles, steps, warm, glob)
    val = r["value"]
    cfg = dict(cfg)
    cfg["workload_timed"] = (f"{r['particles_timed']} particles per step (bounded CPU sample "
                             f"of the {glob}-particle workload)")
    cfg["particles_timed"] = r["particles_timed"]
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
        "steps": steps, "warmup": warm, "ms_per_step": r["sec_per_step"] * 1e3,
        "higher_is_better": True, "scaling": a.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference samplers, seed 0)", "config": cfg,
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": r["cores"], "kind": "port",
                         "sample": r["sample"], "split_s_per_step": r["split_s_per_step"],
                         "extrapolated_full_size": r["extrapolated"]},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def fp64_peak_tflops(torch, dev) -> float:
    from paper_2605_10729_b200 import _native
    lib = _native.load()
    scratch = torch.zeros(8, dtype=torch.float64, device=dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    best = 0.0
    flops = (_native.ctypes.c_double * 3)()
    s = _native.stream_handle(dev)
    for _ in range(6):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        _native.check(lib.pif_probe_fp64(scratch.data_ptr(), sms * 8, 256, 4096, s, flops))
        b.record()
        b.synchronize()
        best = max(best, flops[0] / (a.elapsed_time(b) * 1e-3) / 1e12)
    return best


def load_ncu_traffic():
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def run_b200(a):
    import torch
    import torch.distributed as dist

    import paper_2605_10729_b200 as pb
    from paper_2605_10729_b200.comm import Comm, TorchDistTransport
    from paper_2605_10729_b200.engine import PifEngine
    from paper_2605_10729_b200.samplers import id_slice

    rank, world, local = dist_env()
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else torch.cuda.current_device())
    torch.cuda.set_device(dev)
    cfg, w, per_gpu, glob = workload_config(a, world)
    mk = pb.landau_spec if a.kind == "landau" else pb.penning_spec
    gspec = mk(N=a.N, ppm=max(1, glob // a.N ** 3), dt=a.dt, seed=0)
    plan = pb.make_plan(a.N, gspec.L, a.eps)
    comm = Comm(TorchDistTransport(), rank) if world > 1 else None
    lo, hi = id_slice(glob, rank, world)
    q = gspec.Q_e / glob
    m = abs(gspec.Q_e) / glob
    eng = PifEngine(plan, hi - lo, dev, q=q, m=m, externals=gspec.externals(), dt=a.dt,
                    comm=comm)
    eng.load_sampled(gspec, (lo, hi))

    peak = fp64_peak_tflops(torch, dev)

    # prime solve (strategies.py:290) + warm-up steps
    eng.particle_diag()
    eng.deposit()
    eng.allreduce()
    eng.solve_fields()
    for _ in range(a.warmup):
        eng.step_once()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()

    K = a.steps
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    t_int = [(ev(), ev()) for _ in range(K)]
    t_spr = [(ev(), ev()) for _ in range(K)]
    t_bin = [(ev(), ev()) for _ in range(K)]
    t_fld = [(ev(), ev()) for _ in range(K)]
    t_red = [(ev(), ev()) for _ in range(K)]
    t_mod = [(ev(), ev()) for _ in range(K)]
    start, stop = ev(), ev()
    clocks = ClockSampler(dev.index)
    if rank == 0:
        clocks.start()
        time.sleep(0.3)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    launches0 = eng.launches
    eng.fft_timing(K)
    start.record()
    for i in range(K):
        t_int[i][0].record()
        eng.interp_push()
        t_int[i][1].record()
        t_bin[i][0].record()
        eng.rebin()
        t_bin[i][1].record()
        t_spr[i][0].record()
        eng.spread()
        t_spr[i][1].record()
        t_mod[i][0].record()
        eng.modes()
        t_mod[i][1].record()
        t_red[i][0].record()
        eng.allreduce()
        t_red[i][1].record()
        t_fld[i][0].record()
        eng.solve_fields()
        t_fld[i][1].record()
    stop.record()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clk = clocks.stop() if rank == 0 else None
    launches = eng.launches - launches0
    d2z_ms, z2d_ms = eng.fft_times()
    eng.fft_timing(0)
    T = start.elapsed_time(stop) * 1e-3
    if world > 1:
        tt = torch.tensor([T], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        T = float(tt[0])
    avg = lambda ts: sum(a_.elapsed_time(b_) for a_, b_ in ts) / len(ts) * 1e-3  # noqa: E731
    s_int, s_spr, s_bin, s_fld, s_red = avg(t_int), avg(t_spr), avg(t_bin), avg(t_fld), avg(t_red)
    s_mod = avg(t_mod)
    value = glob * K / T
    f_interp = 6 * w ** 3 + w ** 2
    f_spread = 2 * w ** 3 + w ** 2
    f_step = 8 * w ** 3 + 2 * w ** 2
    achieved = per_gpu * f_interp / s_int / 1e12
    traffic = load_ncu_traffic()
    tr = traffic.get(f"interp_w{w}_ppg{per_gpu}")
    roofline = {
        "bound": "tensor", "pipe": "fp64: DMMA (mma.sync m8n8k4 f64 tensor cores) and DFMA "
                                  "share one ~37 TF/s pipe on B200",
        "kernel": (f"interp_mma_kernel<{w}, 1>" if w <= 8 else f"interp_ring_kernel<{w}, 1>")
                  + " (fused gather + Boris push)",
        "weight_cache": bool(eng.weight_cache),
        "weight_cache_note": "the spread keeps its window weights (192 B/particle) and the next "
                             "gather, at the same positions, loads them instead of evaluating "
                             "them; algorithmic flops are unchanged (weights are not counted)",
        "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
        "frac_vs_nominal_40tf": achieved / 40.0,
        "traffic": tr,
        "peak_source": "fp64 peak measured live in this run by the DFMA probe (pif_probe_fp64; "
                       "DMMA measured equal, profiles/r01_dmma_probe.txt); MEASURED_PEAKS.json "
                       "has HBM and bf16 only; HBM peak from MEASURED_PEAKS.json",
        "algorithmic_flops_per_particle": {"interp": f_interp, "spread": f_spread,
                                           "step": f_step},
        "spread": {"achieved": per_gpu * f_spread / s_spr / 1e12,
                   "frac": per_gpu * f_spread / s_spr / 1e12 / peak},
        "step_fp64_frac": (per_gpu * f_step / (T / K) / 1e12) / peak,
        "hbm_frac_step": None,
        "stage_ms": {"interp_push": s_int * 1e3, "bin": s_bin * 1e3, "spread": s_spr * 1e3,
                     "modes": s_mod * 1e3, "d2z": d2z_ms, "truncate": s_mod * 1e3 - (d2z_ms or 0.0),
                     "allreduce": s_red * 1e3, "fields": s_fld * 1e3, "z2d": z2d_ms,
                     "poisson_guard_pad": s_fld * 1e3 - (z2d_ms or 0.0)},
        "stage_notes": "CUDA events on the launching stream, averaged over the K timed steps; "
                       "d2z / z2d are the cuFFT execs alone (native event pairs around "
                       "cufftExecD2Z / cufftExecZ2D, pif_fft_timing); modes = d2z + truncate/"
                       "deconvolve kernel; fields = finish_deposit+Poisson+energy+guard+pad "
                       "kernels + z2d",
    }
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm = float(json.load(f)["hbm_gbs"])
        roofline["hbm_frac_step"] = per_gpu * 120 / (T / K) / 1e9 / hbm
    except (OSError, KeyError, ValueError):
        pass

    # end to end through the public API with host buffers
    e2e = None
    if not a.no_e2e:
        e2e = run_e2e(a, eng, torch, dist, world, per_gpu, glob, dev)

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        r = cpu_reference_run(a, a.cpu_particles, a.cpu_steps, 0, glob)
        cpu = {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "port",
               "sample": r["sample"], "particles_timed": r["particles_timed"],
               "split_s_per_step": r["split_s_per_step"],
               "extrapolated_full_size": r["extrapolated"]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": a.warmup, "ms_per_step": T / K * 1e3, "higher_is_better": True,
            "scaling": a.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: the reference's own seed-0 ensemble (bench.py Philox "
                    "streams, Landau inverse-CDF / Penning rejection Gaussian, N(0,1) "
                    "velocities) regenerated in HBM by the pif_sample_* kernels",
            "config": cfg, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clk,
        }
        emit(line)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def pin_near_gpu(torch, dev):
    """Move this rank onto the host CPUs local to its GPU (sysfs local_cpulist
    of the GPU's PCI function) while the pinned staging is allocated, so its
    pages land on the GPU's NUMA node and the copies do not cross sockets (the
    caller restores the affinity).  Returns the CPU list (None when the
    topology is not visible).  PIF_E2E_NUMA=0 skips it."""
    if os.environ.get("PIF_E2E_NUMA", "1") != "1":
        return None
    try:
        pr = torch.cuda.get_device_properties(dev)
        bdf = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bdf}/local_cpulist") as f:
            spec = f.read().strip()
        cpus = set()
        for part in spec.split(","):
            lo_, _, hi_ = part.partition("-")
            cpus.update(range(int(lo_), int(hi_ or lo_) + 1))
        if cpus and cpus != set(range(os.cpu_count() or 0)):
            os.sched_setaffinity(0, cpus)
            return spec
        return None
    except Exception:  # noqa: BLE001 - topology not visible: leave placement alone
        return None


def run_e2e(a, eng, torch, dist, world, per_gpu, glob, dev):
    """pif_step-style use with host (pinned) particle arrays in id order (the
    reference's ParticleEnsemble layout) through PifEngine.run_host: per step
    H2D of x, v (ids implied by position), fused load + bin, spread, D2Z,
    allreduce, fields, gather+push writing x, v in id order, D2H of x, v and
    the field energy.  Every rank of the node pins 96 B per particle; if the
    host cannot hold that the line says so instead of failing the run."""
    M = eng.count
    need = 96 * M * int(os.environ.get("LOCAL_WORLD_SIZE", world))
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:  # noqa: BLE001
        avail = None
    if avail is not None and need > 0.8 * avail:
        return {"value": None, "unit": UNIT, "h2d_bytes_per_step": M * 48 * world,
                "d2h_bytes_per_step": (M * 48 + 8) * world,
                "skipped": f"host memory: {need / 1e9:.0f} GB pinned needed, "
                           f"{avail / 1e9:.0f} GB available"}
    lo = int(eng.parts.ids[eng.parts.cur][:M].min())
    cpus0 = os.sched_getaffinity(0)
    numa = pin_near_gpu(torch, dev)
    xh = torch.empty((M, 3), dtype=torch.float64, pin_memory=True)
    vh = torch.empty((M, 3), dtype=torch.float64, pin_memory=True)
    os.sched_setaffinity(0, cpus0)      # pages are placed; the CPU arm keeps every core
    xd, vd = eng.to_id_order(id0=lo)
    xh.copy_(xd)
    vh.copy_(vd)
    del xd, vd

    K = max(1, a.e2e_steps if a.e2e_steps is not None else min(a.steps, 10))
    wh = torch.empty(K, dtype=torch.float64, pin_memory=True)
    eng.run_host(xh, vh, lo, 1, energy_out=wh)       # warm-up (allocates the staging)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    eng.run_host(xh, vh, lo, K, energy_out=wh)
    e.record()
    torch.cuda.synchronize(dev)
    T = s.elapsed_time(e) * 1e-3
    if os.environ.get("PIF_E2E_TRACE") == "1":   # per-step marks to stderr (diagnosis)
        tr = []
        eng.run_host(xh, vh, lo, 4, energy_out=wh, trace=tr)
        torch.cuda.synchronize(dev)
        for i, evs in enumerate(tr):
            print("e2e trace step", i, " ".join(f"{evs[0].elapsed_time(x):.1f}" for x in evs[:7]),
                  file=sys.stderr)
    if world > 1:
        tt = torch.tensor([T], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        T = float(tt[0])
    return {"value": glob * K / T, "unit": UNIT, "h2d_bytes_per_step": M * 48 * world,
            "d2h_bytes_per_step": (M * 48 + 8) * world, "steps": K, "host_cpus": numa,
            "api": "PifEngine.run_host (pif_step-style): per step H2D x,v (pinned, id order) -> "
                   "fused AoS load/wrap/keys + bin -> deposit -> allreduce -> solve_fields -> "
                   "gather+push (also writing x,v in id order) -> D2H x,v,W; step s's D2H and "
                   "step s+1's H2D chunk-pipelined"}


_JSON_OUT = None


def emit(line: dict) -> None:
    """The one JSON line, on the original stdout."""
    out = _JSON_OUT or sys.stdout
    print(json.dumps(line), file=out, flush=True)


def main():
    # stdout carries exactly the JSON line: anything else written to fd 1
    # (NCCL's version banner under torchrun, library chatter) goes to stderr
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_b200(a)


if __name__ == "__main__":
    main()
