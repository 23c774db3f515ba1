"""Wavefront timeline of one Lorenzo launch (needs the -DLZ7_TIMING build via
FZB_SO): per-tile claim / first-step / end times, so the single-field time
splits into per-tile work, dependency waits and SM idling.
    FZB_SO=.../libfzb200_tim.so python scripts/lz_timeline.py 512x512x512 [enc|dec]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2509_20563_b200.device import default_engine, _p, pad3
from paper_2509_20563_b200 import data

dims = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "512x512x512").split("x"))
eng = default_engine(); L = eng.lib
lib = ctypes.CDLL(os.environ["FZB_SO"])
x = data.smooth_trig_device(dims, 0); n = x.numel()
eb = torch.tensor([1e-3 * float(x.max() - x.min())], dtype=torch.float64, device="cuda")
n0, n1, n2 = pad3(dims)
codes = torch.zeros(n + 16, dtype=torch.int16, device="cuda")
bitmap = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
ws = torch.zeros(L.fzb_lorenzo_workspace_bytes(n0, n1, n2), dtype=torch.uint8, device="cuda")
buf = np.zeros((1 << 16, 4), np.uint64)
for dec in (0, 1):
    for _ in range(3):
        if dec == 0:
            L.fzb_lorenzo_encode_f32(_p(x), n0, n1, n2, _p(eb), 512, _p(codes), _p(bitmap), _p(ws), ws.numel(), eng.sp)
        else:
            rec = x.clone()
            L.fzb_lorenzo_decode_f32(_p(codes), _p(bitmap), _p(rec), n0, n1, n2, _p(eb), 512, _p(ws), ws.numel(), eng.sp)
    torch.cuda.synchronize()
    assert lib.fzb_debug_tile_times(buf.ctypes.data_as(ctypes.c_void_p)) == 0
    used = buf[:, 2] > 0
    T = np.nonzero(used)[0]
    t = buf[T].astype(np.float64)
    t0 = t[:, 0].min()
    claim, first, end = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3   # us
    span = end.max()
    work = end - first
    wait = first - claim
    print("dec" if dec else "enc", dims, "tiles", len(T), "span %.1f us" % span,
          "tile work median %.1f us (min %.1f max %.1f)" % (np.median(work), work.min(), work.max()),
          "first-step wait median %.1f us (max %.1f)" % (np.median(wait), wait.max()))
    # concurrency profile: tiles running at time tt
    grid = np.linspace(0, span, 41)
    conc = [int(((first <= g) & (end > g)).sum()) for g in grid]
    claimed = [int(((claim <= g) & (end > g)).sum()) for g in grid]
    print("  running tiles over time:", conc)
    print("  resident (claimed) over time:", claimed)
    print("  sum(work) / span = %.1f tiles busy on average" % (work.sum() / span))
