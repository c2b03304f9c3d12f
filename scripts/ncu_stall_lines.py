"""Per-CUDA-line share of one stall reason from an ncu source export
(--page source --csv --print-source cuda,sass).  usage: ncu_stall_lines.py x.csv REASON [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
reason = sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25


def f(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return 0.0


cur, hdr, agg = None, None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 10 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or r[0] == "":
        continue
    col = next((i for i, h in enumerate(hdr) if h == reason), None)
    if col is None:
        sys.exit(f"no column {reason}; have {[h for h in hdr if h.startswith('stall')][:30]}")
    agg.append((cur, r[0], r[1], f(r[col])))
tot = sum(a[3] for a in agg) or 1
for a in sorted(agg, key=lambda a: -a[3])[:top]:
    print(f"{100 * a[3] / tot:5.1f}%  {a[0]}:{a[1]} {a[2].strip()[:90]}")
