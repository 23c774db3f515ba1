"""One device-resident compress+decompress round trip (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_20563_b200.device import default_engine
from paper_2509_20563_b200.pipeline import get_pipeline
from paper_2509_20563_b200 import data
dims = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "512x512x512").split("x"))
pipe = sys.argv[2] if len(sys.argv) > 2 else "speed"
rel = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-3
spec = get_pipeline(pipe)
x = data.smooth_trig_device(dims, 0) if len(dims) > 1 else data.particle1d_device(dims[0], 0)
eng = default_engine()
out = torch.empty(x.numel(), dtype=torch.float32, device="cuda")
for _ in range(2):
    da = eng.compress(x, dims, 1, rel, pipeline_id=spec.id, predictor=spec.predictor, codec=spec.primary_codec)
    sz = eng.sizes(da)
    eng.decompress_resident(da, sz, rel * (sz["hi"] - sz["lo"]), out)
torch.cuda.synchronize()
print("ok", sz)
