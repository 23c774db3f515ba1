"""A/B timing of the 3D Lorenzo wavefront builds (FZB_SO) on C2 / C1 shapes,
checking codes and reconstructions against a reference run saved by the
first variant (/tmp/lz3d_ref_*.pt)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_20563_b200.device import default_engine, _p, pad3
from paper_2509_20563_b200 import data
eng = default_engine(); L = eng.lib
tag = os.environ.get("FZB_SO", "default").split("/")[-1]
for dims, rel in [((512, 512, 512), 1e-3), ((100, 500, 500), 1e-4)]:
    x = data.smooth_trig_device(dims, 0)
    n = x.numel(); n0, n1, n2 = pad3(dims)
    eb = torch.tensor([rel * float(x.max() - x.min())], dtype=torch.float64, device="cuda")
    codes = torch.zeros(n + 16, dtype=torch.int16, device="cuda")
    bm = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
    ws = torch.zeros(L.fzb_lorenzo_workspace_bytes(n0, n1, n2), dtype=torch.uint8, device="cuda")
    dws = torch.zeros(L.fzb_lorenzo_workspace_bytes(n0, n1, n2), dtype=torch.uint8, device="cuda")
    rec = torch.zeros(n, dtype=torch.float32, device="cuda")
    te, td = [], []
    for it in range(8):
        bm.zero_(); rec.zero_()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        L.fzb_lorenzo_encode_f32(_p(x), n0, n1, n2, _p(eb), 512, _p(codes), _p(bm), _p(ws), ws.numel(), eng.sp)
        e[1].record()
        # outliers: recon must hold their values (scatter from x where flagged)
        flags = ((bm.view(torch.int32).unsqueeze(1) >> torch.arange(32, device="cuda", dtype=torch.int32)) & 1).reshape(-1)[:n].bool()
        rec[flags] = x[flags]
        e2 = torch.cuda.Event(enable_timing=True); e2.record()
        L.fzb_lorenzo_decode_f32(_p(codes), _p(bm), _p(rec), n0, n1, n2, _p(eb), 512, _p(dws), dws.numel(), eng.sp)
        e[2].record(); torch.cuda.synchronize()
        if it >= 2:
            te.append(e[0].elapsed_time(e[1])); td.append(e2.elapsed_time(e[2]))
    ref = f"/tmp/lz3d_ref_{dims[0]}.pt"
    if not os.path.exists(ref):
        torch.save((codes.cpu(), bm.cpu(), rec.cpu()), ref); same = "ref"
    else:
        c0, b0, r0 = torch.load(ref)
        same = bool(torch.equal(c0, codes.cpu()) and torch.equal(b0, bm.cpu()) and torch.equal(r0.view(torch.int32), rec.cpu().view(torch.int32)))
    print(f"{tag:28s} {dims}  enc {min(te):.3f} ms  dec {min(td):.3f} ms  same={same}", flush=True)
