"""Bitshuffle encode/decode micro-benchmark on the C2 code stream (Lorenzo
codes of smooth_trig 512^3, rel 1e-3): kernel times, algorithmic GB/s, and
A/B byte-equality against the non-persistent encoder (FZB_BS_ENC=3)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2509_20563_b200.device import default_engine, _p, pad3
from paper_2509_20563_b200 import data

eng = default_engine(); L = eng.lib
dims = (512, 512, 512)
x = data.smooth_trig_device(dims, 0); n = x.numel()
eb = torch.tensor([1e-3 * float(x.max() - x.min())], dtype=torch.float64, device="cuda")
n0, n1, n2 = pad3(dims)
codes = torch.zeros(n + 16, dtype=torch.int16, device="cuda")
bitmap = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
ws = torch.zeros(L.fzb_lorenzo_workspace_bytes(n0, n1, n2), dtype=torch.uint8, device="cuda")
assert L.fzb_lorenzo_encode_f32(_p(x), n0, n1, n2, _p(eb), 512, _p(codes), _p(bitmap), _p(ws), ws.numel(), eng.sp) == 0
nb = (n + 255) // 256
bm = torch.zeros(nb * 16, dtype=torch.uint8, device="cuda")
pay = torch.zeros(nb * 128, dtype=torch.int32, device="cuda")
nw = torch.zeros(1, dtype=torch.int64, device="cuda")
bws = torch.zeros(L.fzb_bitshuffle_workspace_bytes(n), dtype=torch.uint8, device="cuda")
out = torch.zeros(n + 16, dtype=torch.int16, device="cuda")
st = torch.zeros(1, dtype=torch.int32, device="cuda")
peak = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6545.6) if os.path.exists("MEASURED_PEAKS.json") else 6545.6
res = {}
ref = None
for mode in ("3", "4"):
    os.environ["FZB_BS_ENC"] = mode
    te, td = [], []
    for it in range(8):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        assert L.fzb_bitshuffle_encode(_p(codes), n, _p(bm), _p(pay), _p(nw), _p(bws), bws.numel(), eng.sp) == 0
        e1.record()
        torch.cuda.synchronize()
        words = int(nw.item())
        e1b = torch.cuda.Event(enable_timing=True); e1b.record()
        assert L.fzb_bitshuffle_decode(_p(bm), _p(pay), words, n, 512, _p(out), _p(bws), bws.numel(), _p(st), eng.sp) == 0
        e2.record()
        torch.cuda.synchronize()
        if it >= 2:
            te.append(e0.elapsed_time(e1)); td.append(e1b.elapsed_time(e2))
    got = (bm.clone(), pay[:words].clone(), words)
    if ref is None:
        ref = got
    algo = 2 * n + n // 16 + 4 * words
    res[mode] = {"enc_ms": round(float(np.median(te)), 4), "dec_ms": round(float(np.median(td)), 4),
                 "enc_frac": round(algo / (np.median(te) * 1e-3) / 1e9 / peak, 3),
                 "dec_frac": round(algo / (np.median(td) * 1e-3) / 1e9 / peak, 3),
                 "equal_to_enc3": bool(torch.equal(got[0], ref[0]) and torch.equal(got[1], ref[1]) and got[2] == ref[2]),
                 "roundtrip": bool(torch.equal(out[:n], codes[:n])), "status": int(st.item())}
print(json.dumps(res))
