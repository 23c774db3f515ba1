"""Where the C4 end-to-end step goes: public-API compress / decompress wall
times with their *_with_timing stage splits, plus pinned PCIe bandwidth."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2509_20563_b200 as fz
from paper_2509_20563_b200 import data
n = 280953867
x = data.particle1d_device(n, 0)
xh = torch.empty(n, dtype=torch.float32, pin_memory=True); xh.copy_(x)
f = fz.Field((n,), xh.numpy())
ebs = fz.ErrorBoundSpec(fz.ErrorMode.VALUE_RANGE_RELATIVE, 1e-4)
for _ in range(2):
    a = fz.compress(f, ebs, "default"); r = fz.decompress(fz.parse_archive(fz.archive_buffer(a)))
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter(); a = fz.compress(f, ebs, "default"); t1 = time.perf_counter()
    b = fz.archive_buffer(a); a2 = fz.parse_archive(b); t2 = time.perf_counter()
    r = fz.decompress(a2); t3 = time.perf_counter()
    print(f"compress {1e3*(t1-t0):.1f} ms  buffer+parse {1e3*(t2-t1):.1f} ms  decompress {1e3*(t3-t2):.1f} ms  "
          f"out pinned={torch.from_numpy(r.data).is_pinned()} type={type(r.data).__name__}")
a, tc = fz.compress_with_timing(f, ebs, "default")
r, td = fz.decompress_with_timing(a)
print("compress stages", {k: round(v * 1e3, 2) for k, v in tc.items()})
print("decompress stages", {k: round(v * 1e3, 2) for k, v in td.items()})
h = xh; d = torch.empty(n, dtype=torch.float32, device="cuda"); h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
def t(fn, reps=3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps
gb = 4 * n / 1e9
print(f"pinned H2D {gb / t(lambda: d.copy_(h, non_blocking=True)):.1f} GB/s, D2H {gb / t(lambda: h2.copy_(d, non_blocking=True)):.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
d2 = torch.empty_like(d)
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
print(f"both directions at once {2 * gb / t(both):.1f} GB/s total")
ph = np.empty(n, np.float32)
print(f"host memcpy pinned->pageable {gb / t(lambda: np.copyto(ph, xh.numpy())):.1f} GB/s")
