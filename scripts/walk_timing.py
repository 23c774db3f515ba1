"""Phase breakdown of the 1D Lorenzo walker (needs the -DLZ7_TIMING build via FZB_SO)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2509_20563_b200.device import default_engine, _p
from paper_2509_20563_b200 import data
n = int(sys.argv[1]) if len(sys.argv) > 1 else 280953867
rel = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-4
eng = default_engine(); L = eng.lib
lib = ctypes.CDLL(os.environ["FZB_SO"])
x = data.particle1d_device(n, 0)
eb = torch.tensor([rel * float(x.max() - x.min())], dtype=torch.float64, device="cuda")
codes = torch.zeros(n + 16, dtype=torch.int16, device="cuda")
bitmap = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
ws = torch.zeros(L.fzb_lorenzo_workspace_bytes(1, 1, n), dtype=torch.uint8, device="cuda")
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    L.fzb_lorenzo_encode_f32(_p(x), 1, 1, n, _p(eb), 512, _p(codes), _p(bitmap), _p(ws), ws.numel(), eng.sp)
    e1.record(); torch.cuda.synchronize()
buf = np.zeros(8, np.int64)
lib.fzb_debug_walk_timing(buf.ctypes.data_as(ctypes.c_void_p))
ev = int((codes[:n] != 512).sum()) + int(bitmap.view(torch.uint32).to(torch.int64).bitwise_count().sum()) if hasattr(torch.Tensor, 'bitwise_count') else int((codes[:n] != 512).sum())
print("encode ms", e0.elapsed_time(e1), "events~", ev, "phases (Mcycles): event", buf[0] / 1e6, "interval", buf[1] / 1e6,
      "block-rest", buf[2] / 1e6, "probe+scan", buf[3] / 1e6, "| loop iters", buf[4], "summary loads", buf[5],
      "block scans", buf[6])
