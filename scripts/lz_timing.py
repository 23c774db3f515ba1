"""Per-step cycle breakdown of tile 0's compute warps (needs the -DLZ7_TIMING build via FZB_SO)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2509_20563_b200.device import default_engine, _p, pad3
from paper_2509_20563_b200 import data
dims = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "8x32x512").split("x"))
eng = default_engine(); L = eng.lib
fn = L._lib.fzb_debug_lz_timing if hasattr(L, "_lib") else None
lib = ctypes.CDLL(os.environ["FZB_SO"])
x = data.smooth_trig_device(dims, 0); n = x.numel()
eb = torch.tensor([1e-3 * float(x.max() - x.min())], dtype=torch.float64, device="cuda")
n0, n1, n2 = pad3(dims)
codes = torch.zeros(n + 16, dtype=torch.int16, device="cuda")
bitmap = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
ws = torch.zeros(L.fzb_lorenzo_workspace_bytes(n0, n1, n2), dtype=torch.uint8, device="cuda")
for dec in (0, 1):
    for _ in range(3):
        if dec == 0:
            L.fzb_lorenzo_encode_f32(_p(x), n0, n1, n2, _p(eb), 512, _p(codes), _p(bitmap), _p(ws), ws.numel(), eng.sp)
        else:
            rec = x.clone()
            L.fzb_lorenzo_decode_f32(_p(codes), _p(bitmap), _p(rec), n0, n1, n2, _p(eb), 512, _p(ws), ws.numel(), eng.sp)
    torch.cuda.synchronize()
    buf = np.zeros((8, 1024, 4), np.int64)
    assert lib.fzb_debug_lz_timing(buf.ctypes.data_as(ctypes.c_void_p)) == 0
    for w in range(8):
        st = buf[w]
        valid = st[:, 0] > 0
        if valid.sum() < 20:
            continue
        st = st[valid][16:-16]
        step = np.diff(st[:, 0])
        print("dec" if dec else "enc", "warp", w, "steps", len(st), "cycles/step median", int(np.median(step)),
              "poll", int(np.median(st[:, 1] - st[:, 0])), "shfl+pred", int(np.median(st[:, 2] - st[:, 1])),
              "quant", int(np.median(st[:, 3] - st[:, 2])), "tail", int(np.median(st[1:, 0] - st[:-1, 3])))
