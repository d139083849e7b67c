"""Summarise ncu outputs into profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py launches gpurun_out/launches.csv  > profiles/x_launches.md
  python tools/ncu_summary.py full gpurun_out/prof.ncu-rep      > profiles/x_full.md
  python tools/ncu_summary.py traffic gpurun_out/prof.ncu-rep KEY   (updates profiles/ncu_traffic.json)

The launch list is cold-cache and serialised; only the kernel SHARES of the PIF
step are meaningful (kernels after the last FP64 probe = warm-up + timed steps).
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name):
    n = name.split("(")[0].replace("void ", "")
    n = n.replace("pif::<unnamed>::", "").replace("(anonymous namespace)::", "")
    return n[:70]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    seq = []
    for r in rows[hi + 1:]:
        if len(r) > vi:
            try:
                seq.append((short(r[ki]), float(r[vi].replace(",", ""))))
            except ValueError:
                pass
    last_probe = max(i for i, (n, _) in enumerate(seq) if "dfma_probe" in n)
    step = seq[last_probe + 1:]
    # bench: prime solve, W warm-up steps, K timed steps; count steps by interp launches
    n_steps = sum(1 for n, _ in step if n.startswith("interp_mma_kernel"))
    tot, cnt = defaultdict(float), defaultdict(int)
    for n, v in step:
        tot[n] += v
        cnt[n] += 1
    T = sum(tot.values())
    print(f"# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n")
    print(f"source: {os.path.basename(path)}; {len(step)} launches after the FP64 probe, "
          f"{n_steps} PD steps (prime solve + warm-up + timed)\n")
    print("| kernel | launches | ms / launch | share |")
    print("|---|---:|---:|---:|")
    for n, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"| `{n}` | {cnt[n]} | {v / cnt[n] / 1e6:.3f} | {100 * v / T:.1f}% |")
    print(f"\ntotal {T / 1e6:.2f} ms over {n_steps} steps")


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(out))
    return rows[0], rows[1], rows[2:]


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        # atomics: the spread's REDG.ADD.F64 plane flushes and the push's cell counts
        "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum",
        "lts__t_requests_srcunit_tex_op_red.sum",
        "lts__t_sectors_srcunit_tex_op_red.sum",
        "lts__t_sectors_srcunit_tex_op_red.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum"]


def full(path):
    h, u, rows = raw(path)
    stall = [c for c in h if c.startswith("smsp__pcsamp_warps_issue_stalled")
             and not c.endswith("not_issued")]
    print(f"# ncu --set full summary ({os.path.basename(path)})\n")
    for r in rows:
        print(f"## `{short(r[h.index('Kernel Name')])}`\n")
        print("| metric | value | unit |\n|---|---:|---|")
        for k in KEYS:
            if k in h:
                print(f"| {k} | {r[h.index(k)]} | {u[h.index(k)]} |")
        tot = sum(float(r[h.index(c)] or 0) for c in stall) or 1.0
        top = sorted(((float(r[h.index(c)] or 0), c) for c in stall), reverse=True)[:6]
        print("\nstall samples: " + ", ".join(
            f"{c.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.0f}%"
            for v, c in top) + "\n")


def traffic(path, key, kernel="interp_mma"):
    h, u, rows = raw(path)
    for r in rows:
        if kernel in r[h.index("Kernel Name")]:
            def val(k):
                v = float(r[h.index(k)].replace(",", ""))
                unit = u[h.index(k)]
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
                return v * scale
            b = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
            p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
            d = json.load(open(p)) if os.path.exists(p) else {}
            d[key] = b
            json.dump(d, open(p, "w"), indent=1, sort_keys=True)
            print(key, b)
            return


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        launches(sys.argv[2])
    elif mode == "full":
        full(sys.argv[2])
    elif mode == "traffic":
        traffic(sys.argv[2], sys.argv[3])
