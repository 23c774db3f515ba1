"""Diagnostic: public-API round trips from 1 vs 2 host threads (own CUDA streams)."""
import os, sys, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2509_20563_b200 as fz
from paper_2509_20563_b200 import data
n = int(sys.argv[1]) if len(sys.argv) > 1 else 280953867
x = data.particle1d_device(n, 0)
xh = torch.empty(n, dtype=torch.float32, pin_memory=True); xh.copy_(x)
field = fz.Field((n,), xh.numpy())
ebs = fz.ErrorBoundSpec(fz.ErrorMode.VALUE_RANGE_RELATIVE, 1e-4)
def rt(tag, log):
    t0 = time.perf_counter(); a = fz.compress(field, ebs, "default"); t1 = time.perf_counter()
    p = fz.parse_archive(fz.archive_buffer(a)); t2 = time.perf_counter()
    r = fz.decompress(p); t3 = time.perf_counter()
    log.append((tag, round((t1-t0)*1e3,1), round((t2-t1)*1e3,1), round((t3-t2)*1e3,1)))
    return r
def worker(tag, cnt, log):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(cnt):
            r = rt(tag, log)
log = []
for _ in range(3): rt("serial", log)
print("serial", log[-2:], flush=True)
log = []
ths = [threading.Thread(target=worker, args=(f"T{i}", 3, log)) for i in range(2)]
t0 = time.perf_counter(); [t.start() for t in ths]; [t.join() for t in ths]; dt = time.perf_counter() - t0
print("2 threads total s", round(dt, 3), log, flush=True)
log = []
ths = [threading.Thread(target=worker, args=(f"T{i}", 3, log)) for i in range(2)]
t0 = time.perf_counter(); [t.start() for t in ths]; [t.join() for t in ths]; dt = time.perf_counter() - t0
print("2 threads again total s", round(dt, 3), log, flush=True)
