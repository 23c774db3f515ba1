"""Markdown table of an ncu --set full report: per launch duration, DRAM
traffic, SM / issue / occupancy figures and the top stall reasons.
    python scripts/ncu_table.py report.ncu-rep "title" > out.md"""
import csv, io, subprocess, sys

rep, title = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]


def v(r, k):
    try:
        return float(r[h.index(k)].replace(",", ""))
    except (ValueError, IndexError):
        return float("nan")


def ms(r):
    x = v(r, "gpu__time_duration.sum")
    u = units[h.index("gpu__time_duration.sum")]
    return x / 1e6 if u in ("ns", "nsecond") else (x / 1e3 if u in ("us", "usecond") else x)


def mb(r, k):
    x = v(r, k)
    u = units[h.index(k)]
    return x / 1e6 if u == "byte" else (x / 1e3 if u == "Kbyte" else (x * 1e3 if u == "Gbyte" else x))


print(f"# {title}\n")
print("| kernel | ms | DRAM read MB | DRAM write MB | DRAM % of peak | SM throughput % | issue active % | warps active % | regs | top stalls (per issue) |")
print("|---|---|---|---|---|---|---|---|---|---|")
for r in rows[2:]:
    name = r[h.index("Kernel Name")].replace("void ", "").split("(")[0].replace("<unnamed>::", "")
    st = sorted(((v(r, k), k.split("stalled_")[1].split("_per")[0]) for k in h
                 if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("_per_issue_active.ratio")),
                reverse=True)[:3]
    print(f"| `{name}` | {ms(r):.3f} | {mb(r, 'dram__bytes_read.sum'):.1f} | "
          f"{mb(r, 'dram__bytes_write.sum'):.1f} | {v(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
          f"{v(r, 'sm__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
          f"{v(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
          f"{v(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | {v(r, 'launch__registers_per_thread'):.0f} | "
          + ", ".join(f"{n} {x:.2f}" for x, n in st) + " |")
