"""Summarise a GPU session's ncu outputs into profiles/<round>/ (tracked).

    python scripts/summarize_profiles.py gpurun_out/r01d profiles/r01
Reads launches_*.csv (gpu__time_duration.sum lists) and an optional
full_*.ncu-rep raw CSV export (/tmp/raw_<name>.csv made by `ncu -i ... --page raw --csv`).
"""
import csv, json, os, sys
from collections import defaultdict

src, dst = sys.argv[1], sys.argv[2]
os.makedirs(dst, exist_ok=True)
SKIP = ("at::", "at_cuda_detail", "elementwise", "distribution_", "fill_kernel", "arange", "quality_leaf")


def launches(path):
    rows = list(csv.reader(open(path)))
    h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    H = rows[h]
    ki, vi, ui = H.index("Kernel Name"), H.index("Metric Value"), H.index("Metric Unit")
    agg = defaultdict(list)
    for r in rows[h + 1:]:
        if len(r) > vi and not any(s in r[ki] for s in SKIP):
            v = float(r[vi].replace(",", ""))
            unit = r[ui]
            us = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)
            agg[r[ki].split("(")[0].replace("void ", "")[:48]].append(us)
    return agg


md = ["# ncu launch lists (gpu__time_duration.sum, --clock-control none)\n",
      "Cold-cache, serialised per-launch times; shares (not absolutes) compare with bench.py. "
      "Each capture runs 2 round trips (scripts/prof_roundtrip.py) or a 2-step bench; totals below are per round trip.\n"]
for name, title in (("launches_c2.csv", "C2 Speed 512^3 rel 1e-3 (bench.py --steps 2 --warmup 1)"),
                    ("launches_c1.csv", "C1 Default 100x500x500 rel 1e-4 (scripts/prof_roundtrip.py)"),
                    ("launches_c3.csv", "C3 Quality 1800x3600 rel 1e-4 (scripts/prof_roundtrip.py)"),
                    ("launches_c4.csv", "C4 Default particle1d 280953867 rel 1e-4 (scripts/prof_roundtrip.py)")):
    p = os.path.join(src, name)
    if not os.path.exists(p):
        continue
    agg = launches(p)
    # round trips in the capture = launches of the (one-per-round-trip) min/max kernel
    rt = max(1, len(agg.get("<unnamed>::minmax_final_kernel", [1])))
    tot = sum(sum(v) for v in agg.values()) / rt
    md.append(f"\n### {title}\n\n| kernel | us / round trip | share | launches / rt |\n|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))[:20]:
        md.append(f"| `{k}` | {sum(v) / rt:.1f} | {sum(v) / rt / tot:.1%} | {len(v) / rt:g} |")
    md.append(f"| **total** | {tot:.1f} | | |")
open(os.path.join(dst, "launch_summary.md"), "w").write("\n".join(md) + "\n")
print("\n".join(md))
