"""Summarise an ncu launch-list CSV (gpu__time_duration.sum per launch): time share per kernel."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
agg = defaultdict(list)
for r in rows[hdr + 1:]:
    if len(r) > vi:
        agg[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{sum(v)/1e6:9.3f} ms {len(v):4d} launches  avg {sum(v)/len(v)/1e3:9.1f} us  {100*sum(v)/tot:5.1f}%  {k}")
