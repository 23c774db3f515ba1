"""Summarise an `ncu --page source --csv --print-source sass` dump: top
instructions by stall samples, with their dominant stall reasons, and the
annotated window around a given address range.
    python scripts/ncu_src.py src.csv [top_n] [lo_idx hi_idx]"""
import csv, sys

rows = list(csv.reader(open(sys.argv[1])))
sec = int(__import__("os").environ.get("SECTION", "0"))   # which kernel of a multi-kernel dump
starts = [k for k, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
print(rows[starts[sec]][1][:100])
hdr = rows[starts[sec] + 1]
data = rows[starts[sec] + 2:starts[sec + 1]]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "(Not Issued)" not in h]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print("total samples", tot)
agg = {}
for r in data:
    for h in reasons:
        agg[h] = agg.get(h, 0) + int(r[ix[h]] or 0)
print("by reason:", ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]))


def line(k, r):
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    rs = sorted(((int(r[ix[h]] or 0), h[6:]) for h in reasons), reverse=True)[:3]
    return f"{k:5d} {s:6d} {100 * s / tot:5.1f}%  {r[1].strip()[:60]:60s} " + " ".join(f"{n}:{v}" for v, n in rs if v)


if len(sys.argv) > 4:
    lo, hi = int(sys.argv[3]), int(sys.argv[4])
    for k in range(lo, hi):
        print(line(k, data[k]))
else:
    order = sorted(range(len(data)), key=lambda k: -int(data[k][ix["Warp Stall Sampling (All Samples)"]] or 0))
    for k in order[:top]:
        print(line(k, data[k]))
