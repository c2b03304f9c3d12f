"""Write profiles/traffic.json entries from an ncu --set full report of bench.py:
dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernels,
stamped with the sha of the CUDA sources (bench.py reports the figure only while the
kernels are unchanged).  usage: update_traffic.py REP.ncu-rep CONFIG"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

rep, cfg = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
ki, rd, wr = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
units = rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
path = os.path.join(ROOT, "profiles", "traffic.json")
t = json.load(open(path)) if os.path.exists(path) else {}
t.setdefault(cfg, {})
sha = bench.source_sha()
for r in rows[2:]:
    name = r[ki]
    kind = "spread" if "spread" in name else ("interp" if "interp" in name else None)
    if kind is None:
        continue
    b = float(r[rd].replace(",", "")) * scale[units[rd]] + float(r[wr].replace(",", "")) * scale[units[wr]]
    if b != b:  # ncu reported nan for this launch
        print(cfg, kind, "nan (not recorded)", name[:60])
        continue
    t[cfg][kind] = {"bytes": int(b), "src_sha": sha, "kernel": name.split("(")[0][:80]}
    print(cfg, kind, f"{b / 1e9:.2f} GB", name[:60])
t["_source"] = ("ncu --set full --clock-control none: dram__bytes_read.sum + dram__bytes_write.sum "
                "per launch; src_sha = bench.source_sha() of the kernels measured")
json.dump(t, open(path, "w"), indent=1)
