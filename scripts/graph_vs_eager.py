"""Time one C4 round trip eagerly and as graph replays, per half (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_20563_b200 import data
from paper_2509_20563_b200.device import default_engine, graph_engine
from paper_2509_20563_b200.pipeline import get_pipeline
n = int(sys.argv[1]) if len(sys.argv) > 1 else 280953867
preset = sys.argv[2] if len(sys.argv) > 2 else "default"
x = data.particle1d_device(n, 0)
spec = get_pipeline(preset)
kw = dict(pipeline_id=spec.id, predictor=spec.predictor, codec=spec.primary_codec, radius=spec.radius())
out = torch.empty(n, dtype=torch.float32, device="cuda")
for name, eng, comp, dec in [("eager", default_engine(), "compress", "decompress_resident"),
                             ("graph", graph_engine(), "compress_graphed", "decompress_graphed")]:
    for it in range(5):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record(eng.stream)
        da = getattr(eng, comp)(x, (n,), 1, 1e-4, **kw)
        e[1].record(eng.stream)
        sz = eng.sizes(da)
        e[2].record(eng.stream)
        getattr(eng, dec)(da, sz, 1e-4 * (sz["hi"] - sz["lo"]), out)
        e[3].record(eng.stream)
        torch.cuda.synchronize()
        print(name, it, "compress %.3f ms  sizes %.3f  decompress %.3f" % (e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3])), flush=True)
