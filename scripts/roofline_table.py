"""Per-kernel DRAM roofline table from `ncu --page raw --csv` exports of one
round trip per config, plus profiles/traffic.json (DRAM bytes per C-ABI entry
point per launch, the `traffic` of bench.py's roofline).
    python scripts/roofline_table.py gpurun_out/r02q2 profiles/r02"""
import csv, json, os, sys

src, dst = sys.argv[1], sys.argv[2]
PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6540.5
# kernel name prefix -> C-ABI entry point (bench.py's `dom` keys)
ENTRY = {"lz1d_summary2": "fzb_lorenzo1d_prepare_f32", "lz1d_super": "fzb_lorenzo1d_prepare_f32",
         "lz1d_lohi": "fzb_lorenzo1d_prepare_f32", "lz1d_walk3": "fzb_lorenzo1d_walk_f32",
         "hist_flagged": "fzb_histogram_flagged", "v6::lz7_kernel<4, 2, 0>": "fzb_lorenzo_encode_f32",
         "v6::lz7_kernel<8, 1, 0>": "fzb_lorenzo_encode_f32", "v6::lz7_kernel<4, 2, 1>": "fzb_lorenzo_decode_f32",
         "v6::lz7_kernel<8, 1, 1>": "fzb_lorenzo_decode_f32", "lz1d_event": "fzb_lorenzo_decode_f32",
         "lz1d_chain2": "fzb_lorenzo_decode_f32", "lz1d_fill2": "fzb_lorenzo_decode_f32",
         "bs_enc4": "fzb_bitshuffle_encode", "bs_dec": "fzb_bitshuffle_decode", "hf_count": "fzb_huffman_encode_chunks",
         "hf_write2": "fzb_huffman_encode_chunks", "hf_zero": "fzb_huffman_encode_chunks", "hf_sync": "fzb_huffman_decode",
         "hf_write_dec2": "fzb_huffman_decode", "hf_tables": "fzb_huffman_decode", "hist_smem": "fzb_histogram_chunks",
         "minmax": "fzb_minmax_f32", "interp_pass_kernel<0, 0>": "fzb_interp_encode_f32",
         "interp_pass_kernel<1, 0>": "fzb_interp_encode_f32", "interp_pass_kernel<2, 0>": "fzb_interp_encode_f32",
         "interp_pass_kernel<0, 1>": "fzb_interp_decode_f32", "interp_pass_kernel<1, 1>": "fzb_interp_decode_f32",
         "interp_pass_kernel<2, 1>": "fzb_interp_decode_f32", "huffman_build": "fzb_huffman_build",
         "hf_prefill": "fzb_huffman_decode", "anchor_kernel<0>": "fzb_interp_encode_f32",
         "anchor_kernel<1>": "fzb_interp_decode_f32"}


def entry_of(name):
    if name.startswith("interp2d_tile_kernel<"):   # last template argument = DEC
        return "fzb_interp_decode_f32" if name.rstrip(">").endswith("1") else "fzb_interp_encode_f32"
    for pre, ent in ENTRY.items():
        if name.startswith(pre):
            return ent
    return None


def load(path):
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        def v(k):
            i = h.index(k)
            x = float(r[i].replace(",", "")) if r[i] not in ("", "n/a") else float("nan")
            u = units[i]
            if k.startswith("dram__bytes"):
                x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            if k == "gpu__time_duration.sum":
                x *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(u, 1)
            return x
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        out.append(dict(name=name, us=v("gpu__time_duration.sum"), rd=v("dram__bytes_read.sum"),
                        wr=v("dram__bytes_write.sum"),
                        issue=v("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                        warps=v("sm__warps_active.avg.pct_of_peak_sustained_active")))
    return out


md = ["# ncu --set full, one round trip per config (--clock-control none; cold, serialised launches)\n",
      f"DRAM GB/s = (dram__bytes_read + dram__bytes_write) / gpu__time_duration; % of the measured {PEAK:.0f} GB/s copy peak.\n"]
traffic = {"source": f"{src} (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum per launch)", "kernels": {}}
for cfg in ("c4", "c2", "c3"):
    p = os.path.join(src, f"raw_{cfg}.csv")
    if not os.path.exists(p):
        continue
    ks = load(p)
    # prof_roundtrip runs the round trip twice; keep the last launch of every
    # (kernel, occurrence-within-the-trip) -- the warm one where both exist
    seen, half = {}, []
    for k in ks:
        seen[k["name"]] = seen.get(k["name"], 0) + 1
    cnt = {}
    for k in ks:
        cnt[k["name"]] = cnt.get(k["name"], 0) + 1
        per_trip = max(1, seen[k["name"]] // 2) if seen[k["name"]] > 1 else 1
        if seen[k["name"]] == 1 or cnt[k["name"]] > seen[k["name"]] - per_trip:
            half.append(k)
    md.append(f"\n## {cfg}\n\n| kernel | us | DRAM MB | DRAM GB/s | % peak | issue % | warps % |\n|---|---|---|---|---|---|---|")
    per_entry = {}
    for k in half:
        mbytes = (k["rd"] + k["wr"]) / 1e6
        gbs = (k["rd"] + k["wr"]) / (k["us"] * 1e3) if k["us"] > 0 else 0
        md.append(f"| {k['name'][:48]} | {k['us']:.1f} | {mbytes:.1f} | {gbs:.0f} | {100 * gbs / PEAK:.0f} | "
                  f"{k['issue']:.0f} | {k['warps']:.0f} |")
        ent = entry_of(k["name"])
        if ent:
            per_entry[ent] = per_entry.get(ent, 0) + k["rd"] + k["wr"]
    for ent, b in per_entry.items():
        traffic["kernels"][f"{cfg}:{ent}"] = {"bytes": int(b)}
os.makedirs(dst, exist_ok=True)
open(os.path.join(dst, "ncu_full.md"), "w").write("\n".join(md) + "\n")
json.dump(traffic, open(os.path.join("profiles", "traffic.json"), "w"), indent=1)
print("\n".join(md))
