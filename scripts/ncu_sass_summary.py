"""Summarise an ncu --page source (SASS) CSV export: instructions and stall samples
per opcode, plus the hottest SASS lines.  Usage:
  ncu -i rep --page source --csv -k regex:NAME > x.csv ; python scripts/ncu_sass_summary.py x.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r)
h = rows[hi]
si, ie, ws = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[hi + 1:] if len(r) > ie and r[si].strip() and r[ie].replace(",", "").replace(".", "").isdigit()]
f = lambda v: float(v.replace(",", "") or 0)
tot_i = sum(f(r[ie]) for r in data)
tot_s = sum(f(r[ws]) for r in data)
by_op_i, by_op_s = defaultdict(float), defaultdict(float)
for r in data:
    op = r[si].split()[0]
    if op.startswith("@"):
        op = r[si].split()[1]
    op = op.split(".")[0]
    by_op_i[op] += f(r[ie])
    by_op_s[op] += f(r[ws])
print(f"warp instructions {tot_i:.3e}, stall samples {tot_s:.0f}")
for op in sorted(by_op_i, key=lambda o: -by_op_i[o])[:25]:
    print(f"{op:10s} inst {100 * by_op_i[op] / tot_i:5.1f}%  stall {100 * by_op_s[op] / max(tot_s, 1):5.1f}%")
print("--- hottest lines (stall samples)")
for r in sorted(data, key=lambda r: -f(r[ws]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{100 * f(r[ws]) / max(tot_s, 1):5.1f}%  {r[si].strip()[:100]}")
