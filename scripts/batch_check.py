"""compress_batch / decompress_batch_resident vs per-field Engine.compress: identical
archives and reconstructions; timing of F fields in one batch vs F single fields."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2509_20563_b200 import data
from paper_2509_20563_b200.device import default_engine
from paper_2509_20563_b200.pipeline import get_pipeline

dims = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "128x256x256").split("x"))
pipe = sys.argv[2] if len(sys.argv) > 2 else "speed"
Fs = [int(v) for v in (sys.argv[3] if len(sys.argv) > 3 else "1,2,4").split(",")]
rel = 1e-3
spec = get_pipeline(pipe)
eng = default_engine()
n = int(np.prod(dims))
Fmax = max(Fs)
X = torch.stack([data.smooth_trig_device(dims, s) for s in range(Fmax)]).contiguous()
kw = dict(pipeline_id=spec.id, predictor=spec.predictor, codec=spec.primary_codec, radius=spec.radius())

# reference: single fields
ref = []
for f in range(Fmax):
    da = eng.compress(X[f], dims, 1, rel, **kw)
    lo, hi, segs = eng.finish(da)
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    sz = eng.sizes(da)
    eng.decompress_resident(da, sz, rel * (sz["hi"] - sz["lo"]), out)
    torch.cuda.synchronize()
    ref.append(([bytes(p) for _, p in segs], out.clone()))

for F in Fs:
    das = eng.compress_batch(X[:F], dims, 1, rel, **kw)
    szs = eng.sizes_batch(das)
    OUT = torch.empty(F, n, dtype=torch.float32, device="cuda")
    eng.decompress_batch_resident(das, szs, [rel * (z["hi"] - z["lo"]) for z in szs], OUT)
    torch.cuda.synchronize()
    ok = True
    for f in range(F):
        lo, hi, segs = eng.finish(das[f])
        ok &= [bytes(p) for _, p in segs] == ref[f][0]
        ok &= bool(torch.equal(OUT[f].view(torch.int32), ref[f][1].view(torch.int32)))
    # timing: batch vs loop of singles
    def batch():
        d = eng.compress_batch(X[:F], dims, 1, rel, **kw)
        z = eng.sizes_batch(d)
        eng.decompress_batch_resident(d, z, [rel * (q["hi"] - q["lo"]) for q in z], OUT)
    def singles():
        for f in range(F):
            d = eng.compress(X[f], dims, 1, rel, **kw)
            z = eng.sizes(d)
            eng.decompress_resident(d, z, rel * (z["hi"] - z["lo"]), OUT[f])
    res = {}
    for name, fn in (("batch", batch), ("singles", singles)):
        fn(); torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        res[name] = (time.perf_counter() - t0) / 3
    print(f"F={F} identical={ok} batch {res['batch']*1e3:.2f} ms ({F*4*n/res['batch']/1e9:.1f} GB/s)  "
          f"singles {res['singles']*1e3:.2f} ms ({F*4*n/res['singles']/1e9:.1f} GB/s)", flush=True)
