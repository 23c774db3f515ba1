"""Instruction mix per kernel from an ncu report's source page:
    python scripts/ncu_mix.py report.ncu-rep kernel_regex units"""
import csv, io, subprocess, sys

rep, kre, units = sys.argv[1], sys.argv[2], float(sys.argv[3])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kre,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
st = [k for k, r in enumerate(rows) if r and r[0] == "Kernel Name"]
hdr = rows[st[0] + 1]
data = rows[st[0] + 2:(st[1] if len(st) > 1 else len(rows))]
ix = {h: i for i, h in enumerate(hdr)}
tot, ops = 0, {}
for r in data:
    ex = int(r[ix["Instructions Executed"]] or 0)
    t = r[1].strip().split()
    if not t:
        continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    ops[op] = ops.get(op, 0) + ex
    tot += ex
print(rows[st[0]][1][:80], "| warp-instr per unit %.1f" % (tot / units))
print("  " + ", ".join(f"{k} {v / units:.1f}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:16]))
