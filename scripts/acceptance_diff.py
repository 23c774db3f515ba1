"""Replay fzpipe's acceptance criterion 1 (200 randomised triples,
test_acceptance.py:99-130) through fzpipe's CPU path AND this package's GPU
path, and print every triple whose archive or reconstruction differs.
Needs baseline/_ref (scripts/install_reference.sh) and a GPU."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(0, ROOT)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/fzpipe_numba_cache")

import fzpipe  # noqa: E402
from fzpipe.data import SyntheticSpec, generate  # noqa: E402

import paper_2509_20563_b200 as fz  # noqa: E402

PRESETS = ["default", "speed", "quality"]
EBS = [1e-6, 1e-4, 1e-2]
rng = np.random.default_rng(2024)
dims_pool = [(37,), (1000,), (4096,), (1 << 17,), (16, 100), (33, 31), (65, 65), (128, 96), (512, 512),
             (8, 9, 10), (17, 19, 23), (32, 40, 48), (64, 64, 64)]
kinds = ["smooth_trig", "filtered_noise", "piecewise_constant"]
bad = 0
for i in range(200):
    preset = PRESETS[i % 3]
    eb = EBS[(i // 3) % 3]
    dims = (128, 128, 128) if i < 3 else dims_pool[int(rng.integers(0, len(dims_pool)))]
    kind = kinds[int(rng.integers(0, len(kinds)))]
    params = {}
    if kind == "filtered_noise":
        params["width"] = str(int(rng.integers(1, 5)))
    if kind == "piecewise_constant" and len(dims) == 1 and rng.integers(0, 2):
        kind = "particle1d"
        params = {}
    seed = int(rng.integers(0, 10**6))
    f = generate(SyntheticSpec(kind, dims, seed, params))
    spec = fzpipe.ErrorBoundSpec(fzpipe.ErrorMode.VALUE_RANGE_RELATIVE, eb)
    want = fzpipe.serialize_archive(fzpipe.compress(f, spec, preset))
    got = fz.serialize_archive(fz.compress(fz.Field(f.dims, f.data), fz.ErrorBoundSpec(
        fz.ErrorMode.VALUE_RANGE_RELATIVE, eb), preset))
    rw = fzpipe.decompress(fzpipe.parse_archive(want)).data
    rg = fz.decompress(fz.parse_archive(got)).data
    if want != got or rw.tobytes() != rg.tobytes():
        bad += 1
        first = next((k for k in range(min(len(want), len(got))) if want[k] != got[k]), None)
        print(f"#{i} {preset} eb={eb} dims={dims} kind={kind} params={params} seed={seed}: "
              f"len {len(want)} vs {len(got)}, first byte diff {first}, "
              f"recon equal {rw.tobytes() == rg.tobytes()}, max|ours-x| {np.max(np.abs(rg.astype(np.float64) - f.data)):.4g}",
              flush=True)
print("mismatches:", bad)
