"""Aggregate an ncu source-page CSV (SASS view) by opcode: executed warp
instructions and stall samples.  usage: ncu -i rep --page source --csv
--kernel-name regex:K | python tools/sass_hist.py"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(sys.stdin))
hdr = rows[1] if rows[0][0] == "Kernel Name" else rows[0]
start = 2 if rows[0][0] == "Kernel Name" else 1
si, ni, ei = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
ex = defaultdict(int)
st = defaultdict(int)
tot_e = tot_s = 0
for r in rows[start:]:
    if len(r) <= ei:
        continue
    src = r[si].strip()
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", src)
    if not m:
        continue
    op = m.group(2) + (m.group(3) or "")
    op = re.sub(r"\.(E|STRONG\.GPU|RN|SYS|CONSTANT)\b", "", op)
    if not (r[ei] or "0").isdigit():
        continue
    e = int(r[ei] or 0)
    s = int(r[ni] or 0)
    ex[op] += e
    st[op] += s
    tot_e += e
    tot_s += s
print(f"total warp instructions {tot_e:.4g}, stall samples {tot_s}")
for op, e in sorted(ex.items(), key=lambda kv: -kv[1])[:int(sys.argv[1]) if len(sys.argv) > 1 else 30]:
    print(f"{op:28s} {e:14d} {100*e/tot_e:6.2f}%   samples {100*st[op]/max(tot_s,1):6.2f}%")
