"""Huffman codebook build micro-benchmark: device time of fzb_huffman_build
on a C1-like histogram (Lorenzo codes of smooth_trig 100x500x500, rel 1e-4)
and a few synthetic ones."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2509_20563_b200.device import default_engine, _p
eng = default_engine(); L = eng.lib
rng = np.random.default_rng(0)
cases = {"c1like_128": np.round(np.abs(rng.normal(0, 20, 128))).astype(np.uint64) + 1,
         "geo_79": rng.geometric(0.1, 79).astype(np.uint64),
         "ties_200": rng.integers(1, 4, 200).astype(np.uint64),
         "wide_600": rng.geometric(0.01, 600).astype(np.uint64),
         "wide_1000": rng.geometric(0.005, 1000).astype(np.uint64),
         "flat_1024": rng.integers(1000, 2000, 1024).astype(np.uint64)}
for name, used in cases.items():
    bins = np.zeros(1024, np.uint64)
    bins[rng.choice(1024, used.size, replace=False)] = used
    d_bins = torch.from_numpy(bins.view(np.int64)).cuda()
    lengths = torch.zeros(1024, dtype=torch.uint8, device="cuda")
    cw = torch.zeros(1024, dtype=torch.int32, device="cuda")
    bc = torch.zeros(1, dtype=torch.int64, device="cuda")
    ws = torch.zeros(L.fzb_huffman_build_workspace_bytes(1024), dtype=torch.uint8, device="cuda")
    ts = []
    for it in range(12):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        assert L.fzb_huffman_build(_p(d_bins), 1024, _p(lengths), _p(cw), _p(bc), _p(ws), ws.numel(), eng.sp) == 0
        e1.record()
        torch.cuda.synchronize()
        if it >= 2:
            ts.append(e0.elapsed_time(e1) * 1e3)
    print(name, "build us median %.1f min %.1f" % (np.median(ts), np.min(ts)))
    if os.environ.get("FZB_SO"):   # -DLZ7_TIMING build: cycle stamps of the single-warp path
        import ctypes
        dbg = ctypes.CDLL(os.environ["FZB_SO"])
        buf = np.zeros(8, np.int64)
        dbg.fzb_debug_hf_build(buf.ctypes.data_as(ctypes.c_void_p))
        d = np.diff(buf[:6])
        print("   cycles: sort", d[0], "levels", d[1], "prefixes", d[2], "lengths", d[3], "codewords", d[4],
              "fixed point at level", buf[7])

