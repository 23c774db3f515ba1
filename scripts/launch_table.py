"""Per-kernel time per round trip from ncu launch lists (gpu__time_duration.sum).
    python scripts/launch_table.py gpurun_out/X/launches_c4.csv [runs=2]"""
import csv, sys
from collections import defaultdict
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rows = list(csv.reader(open(sys.argv[1])))
h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
H = rows[h]
ki, vi, ui = H.index("Kernel Name"), H.index("Metric Value"), H.index("Metric Unit")
agg = defaultdict(list)
for r in rows[h + 1:]:
    if "at::" in r[ki] or "at_cuda" in r[ki]:
        continue
    v = float(r[vi].replace(",", "")); u = r[ui]
    us = v / 1e3 if u in ("ns", "nsecond") else (v * 1e3 if u in ("ms", "msecond") else v)
    agg[r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")[:50]].append(us)
tot = 0
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    s = sum(v) / runs
    tot += s
    print(f"{s:9.1f} us  x{len(v) // runs:3d}  {k}")
print(f"{tot:9.1f} us  total (our kernels, per round trip)")
