"""One Lorenzo encode + decode launch on a shape (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_20563_b200.device import default_engine, _p, pad3
from paper_2509_20563_b200 import data
dims = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "8x32x512").split("x"))
eng = default_engine(); L = eng.lib
x = data.smooth_trig_device(dims, 0); n = x.numel()
eb = torch.tensor([1e-3 * float(x.max() - x.min())], dtype=torch.float64, device="cuda")
n0, n1, n2 = pad3(dims)
codes = torch.zeros(n + 16, dtype=torch.int16, device="cuda")
bitmap = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
ws = torch.zeros(L.fzb_lorenzo_workspace_bytes(n0, n1, n2), dtype=torch.uint8, device="cuda")
recon = x.clone()
for _ in range(int(os.environ.get("REPS", "1"))):
    bitmap.zero_()
    assert L.fzb_lorenzo_encode_f32(_p(x), n0, n1, n2, _p(eb), 512, _p(codes), _p(bitmap), _p(ws), ws.numel(), eng.sp) == 0
    recon.copy_(x)
    assert L.fzb_lorenzo_decode_f32(_p(codes), _p(bitmap), _p(recon), n0, n1, n2, _p(eb), 512, _p(ws), ws.numel(), eng.sp) == 0
torch.cuda.synchronize()
print("maxerr/eb", float((recon - x).abs().max() / eb))
