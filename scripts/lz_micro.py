"""Micro-benchmark of the Lorenzo wavefront kernels on assorted shapes
(per-step latency = single-tile time / steps)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2509_20563_b200.device import default_engine, _p, pad3
from paper_2509_20563_b200 import data

eng = default_engine()
L = eng.lib
shapes = [(8, 32, 512), (64, 32, 512), (8, 512, 512), (512, 512, 512), (100, 500, 500), (1, 1800, 3600)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in s.split("x")) for s in sys.argv[1:]]
res = {}
for dims in shapes:
    n = int(np.prod(dims))
    x = data.smooth_trig_device(dims, 0)
    lo, hi = float(x.min()), float(x.max())
    eb = torch.tensor([1e-3 * (hi - lo)], dtype=torch.float64, device="cuda")
    codes = torch.empty(n + 16, dtype=torch.int16, device="cuda")
    bitmap = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
    n0, n1, n2 = pad3(dims)
    ws = torch.empty(L.fzb_lorenzo_workspace_bytes(n0, n1, n2), dtype=torch.uint8, device="cuda")
    recon = torch.empty(n, dtype=torch.float32, device="cuda")
    times = {"enc": [], "dec": []}
    for it in range(6):
        bitmap.zero_()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        L.fzb_lorenzo_encode_f32(_p(x), n0, n1, n2, _p(eb), 512, _p(codes), _p(bitmap), _p(ws), ws.numel(), eng.sp)
        e1.record()
        L.fzb_lorenzo_decode_f32(_p(codes), _p(bitmap), _p(recon), n0, n1, n2, _p(eb), 512, _p(ws), ws.numel(), eng.sp)
        e2.record()
        torch.cuda.synchronize()
        if it:
            times["enc"].append(e0.elapsed_time(e1)); times["dec"].append(e1.elapsed_time(e2))
    ok = bool((recon - x).abs().max().item() <= eb.item())
    r = {k: round(float(np.median(v)), 4) for k, v in times.items()}
    r["ok"] = ok
    r["gbs_enc"] = round(4 * n / r["enc"] / 1e6, 1)
    res["x".join(map(str, dims))] = r
    print(dims, r, flush=True)
print(json.dumps(res))
