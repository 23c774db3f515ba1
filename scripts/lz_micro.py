"""Micro-benchmark + A/B bit-exactness of the Lorenzo wavefront kernels
(v6 register wavefront vs v4 barrier wavefront, FZB_LORENZO=4)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2509_20563_b200.device import default_engine, _p, pad3
from paper_2509_20563_b200 import data

eng = default_engine()
L = eng.lib
shapes = [(8, 32, 512), (64, 32, 512), (8, 512, 512), (512, 512, 512), (100, 500, 500), (1, 1800, 3600), (37, 45, 67)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in s.split("x")) for s in sys.argv[1:]]
res = {}


def run(impl, x, dims, eb, reps=6):
    os.environ["FZB_LORENZO"] = impl
    n = x.numel()
    n0, n1, n2 = pad3(dims)
    codes = torch.zeros(n + 16, dtype=torch.int16, device="cuda")
    bitmap = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
    ws = torch.zeros(L.fzb_lorenzo_workspace_bytes(n0, n1, n2), dtype=torch.uint8, device="cuda")
    recon = torch.empty(n, dtype=torch.float32, device="cuda")
    times = {"enc": [], "dec": []}
    for it in range(reps):
        bitmap.zero_()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        rc = L.fzb_lorenzo_encode_f32(_p(x), n0, n1, n2, _p(eb), 512, _p(codes), _p(bitmap), _p(ws), ws.numel(), eng.sp)
        e1.record()
        # outlier values pre-scattered (what fzb_outlier_scatter does)
        recon.copy_(x)
        e1b = torch.cuda.Event(enable_timing=True); e1b.record()
        rc2 = L.fzb_lorenzo_decode_f32(_p(codes), _p(bitmap), _p(recon), n0, n1, n2, _p(eb), 512, _p(ws), ws.numel(), eng.sp)
        e2.record()
        torch.cuda.synchronize()
        assert rc == 0 and rc2 == 0, (rc, rc2)
        if it:
            times["enc"].append(e0.elapsed_time(e1)); times["dec"].append(e1b.elapsed_time(e2))
    return codes[:n].clone(), bitmap.clone(), recon.clone(), times


for dims in shapes:
    n = int(np.prod(dims))
    x = data.smooth_trig_device(dims, 0)
    lo, hi = float(x.min()), float(x.max())
    eb = torch.tensor([1e-3 * (hi - lo)], dtype=torch.float64, device="cuda")
    r = {}
    out = {}
    for impl in ("6", "4"):
        c, bm, rec, t = run(impl, x, dims, eb)
        out[impl] = (c, bm, rec)
        r["enc" + impl] = round(float(np.median(t["enc"])), 4)
        r["dec" + impl] = round(float(np.median(t["dec"])), 4)
    r["codes_eq"] = bool(torch.equal(out["6"][0], out["4"][0]))
    r["bitmap_eq"] = bool(torch.equal(out["6"][1], out["4"][1]))
    r["recon_eq"] = bool(torch.equal(out["6"][2].view(torch.int32), out["4"][2].view(torch.int32)))
    r["ok"] = bool((out["6"][2] - x).abs().max().item() <= eb.item())
    r["gbs_enc6"] = round(4 * n / r["enc6"] / 1e6, 1)
    res["x".join(map(str, dims))] = r
    print(dims, r, flush=True)
print(json.dumps(res))
