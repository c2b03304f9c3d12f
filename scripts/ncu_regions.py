"""Group consecutive SASS lines of an ncu source CSV into regions with equal execution
counts and print instructions per region (a poor man's basic-block profile)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
ncta = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r)
h = rows[hi]; si = h.index("Source"); ie = h.index("Instructions Executed")
ws = h.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[hi + 1:] if len(r) > ie and r[ie].replace(",", "").replace(".", "").isdigit()]
f = lambda v: float(v.replace(",", "") or 0)
tot = sum(f(r[ie]) for r in data); tots = sum(f(r[ws]) for r in data)
regions = []
for k, r in enumerate(data):
    c = f(r[ie])
    if regions and abs(regions[-1][2] - c) <= 0.02 * max(c, 1):
        regions[-1][1] = k; regions[-1][3] += c; regions[-1][4] += f(r[ws])
    else:
        regions.append([k, k, c, c, f(r[ws])])
for a, b, c, s, st in regions:
    if s / tot > 0.01 or st / tots > 0.02:
        print(f"[{a:4d}-{b:4d}] n={b-a+1:3d} x {c/ncta:9.1f}/cta  inst {100*s/tot:5.1f}%  stall {100*st/tots:5.1f}%  | {data[a][si].strip()[:50]} .. {data[b][si].strip()[:40]}")
