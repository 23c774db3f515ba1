"""cProfile of the public-API round trip (compress(Field) -> Archive -> decompress)."""
import cProfile, io, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2509_20563_b200 as fz
from paper_2509_20563_b200 import data
from paper_2509_20563_b200.core import ErrorBoundSpec, ErrorMode, Field
dims = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "512x512x512").split("x"))
pipe = sys.argv[2] if len(sys.argv) > 2 else "speed"
rel = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-3
x = data.smooth_trig_device(dims, 0)
n = x.numel()
xh = torch.empty(n, dtype=torch.float32, pin_memory=True); xh.copy_(x)
f = Field(dims, xh.numpy())
ebs = ErrorBoundSpec(ErrorMode.VALUE_RANGE_RELATIVE, rel)
for _ in range(2):
    a = fz.compress(f, ebs, pipe); r = fz.decompress(a)
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter(); a, tc = fz.compress_with_timing(f, ebs, pipe); t1 = time.perf_counter()
    r, td = fz.decompress_with_timing(a); t2 = time.perf_counter()
    print(f"compress {1e3*(t1-t0):.1f} ms {tc}  decompress {1e3*(t2-t1):.1f} ms {td}")
pr = cProfile.Profile(); pr.enable()
a = fz.compress(f, ebs, pipe); r = fz.decompress(a)
pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25); print(s.getvalue())
