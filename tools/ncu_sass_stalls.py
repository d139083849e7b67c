"""Aggregate an `ncu --page source --csv --print-source sass` export by opcode
and by instruction index range (for reading stall hot spots of one kernel).

  ncu -i rep --page source --csv --print-source sass -k regex:NAME > k.csv
  python tools/ncu_sass_stalls.py k.csv [--ranges STEP]
"""
import csv
import re
import sys
from collections import defaultdict


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
    h = rows[hi]
    out = []
    for r in rows[hi + 1:]:
        if len(r) != len(h):
            continue
        out.append(dict(zip(h, r)))
    return h, out


def num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return 0.0


def opcode(src):
    return re.sub(r"^@!?U?P\w+\s+", "", src.strip()).split(" ")[0].split(".")[0]


def main():
    h, rows = load(sys.argv[1])
    stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    tot = sum(num(r["Warp Stall Sampling (All Samples)"]) for r in rows)
    by_op = defaultdict(lambda: defaultdict(float))
    for r in rows:
        op = opcode(r["Source"])
        by_op[op]["samples"] += num(r["Warp Stall Sampling (All Samples)"])
        by_op[op]["inst"] += num(r["Instructions Executed"])
        for c in stalls:
            by_op[op][c] += num(r[c])
    print(f"total samples {tot:.0f}")
    print(f"{'op':12s} {'samp%':>6s} {'inst(M)':>9s}  top stalls")
    for op, d in sorted(by_op.items(), key=lambda kv: -kv[1]["samples"])[:25]:
        top = sorted(((c[6:], d[c]) for c in stalls), key=lambda kv: -kv[1])[:4]
        ts = ", ".join(f"{n} {v / max(1, d['samples']) * 100:.0f}%" for n, v in top if v > 0)
        print(f"{op:12s} {d['samples'] / tot * 100:6.1f} {d['inst'] / 1e6:9.1f}  {ts}")
    if "--ranges" in sys.argv:
        k = sys.argv.index("--ranges")
        step = int(sys.argv[k + 1]) if len(sys.argv) > k + 1 else 64
        print("\nby instruction index range")
        for i in range(0, len(rows), step):
            chunk = rows[i:i + step]
            s = sum(num(r["Warp Stall Sampling (All Samples)"]) for r in chunk)
            inst = sum(num(r["Instructions Executed"]) for r in chunk)
            if s < 0.002 * tot:
                continue
            ops = defaultdict(int)
            for r in chunk:
                ops[opcode(r["Source"])] += 1
            top = ", ".join(f"{a}:{b}" for a, b in sorted(ops.items(), key=lambda kv: -kv[1])[:5])
            st = defaultdict(float)
            for r in chunk:
                for c in stalls:
                    st[c[6:]] += num(r[c])
            tops = ", ".join(f"{a} {b / max(1, s) * 100:.0f}%" for a, b in
                             sorted(st.items(), key=lambda kv: -kv[1])[:3])
            print(f"[{i:5d}] samp {s / tot * 100:5.1f}% inst {inst / 1e6:8.1f}M | {top} | {tops}")


if __name__ == "__main__":
    main()
