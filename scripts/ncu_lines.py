"""Per-CUDA-line instruction and stall-sample shares from an ncu source export
(ncu -i rep --page source --csv --print-source cuda,sass -k regex:K > x.csv).
usage: python scripts/ncu_lines.py x.csv [npoints] [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))


def f(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return 0.0


cur, agg = None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] in ("Line No", ""):
        continue
    agg.append((cur, r[0], r[1], f(r[4]), f(r[7])))
ti = sum(a[4] for a in agg) or 1
ts = sum(a[3] for a in agg) or 1
npts = float(sys.argv[2]) if len(sys.argv) > 2 else 0
if npts:
    print(f"{ti / npts:.1f} warp instructions per point")
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
for a in sorted(agg, key=lambda a: -a[4])[:top]:
    per = f" {a[4] / npts:5.2f}/pt" if npts else ""
    print(f"{100 * a[4] / ti:5.1f}% inst{per} {100 * a[3] / ts:5.1f}% stall  {a[0]}:{a[1]} {a[2].strip()[:80]}")
