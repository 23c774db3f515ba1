"""Workspace reuse across shapes: one Engine runs the v7 wavefront (n2 % 4 ==
0), the v4 wavefront (other 3D/2D shapes) and the 1D walker on the SAME
Lorenzo workspaces, interleaved, and every archive and reconstruction must
still equal the oracle's.  Regression for the round-2 finding (fzpipe's own
test_acceptance.py criterion 1 under the plugin): a v4 or 1D call reset the
v7 launch epoch / left small integers where the next shape's LL faces live,
so a later v7 launch accepted stale halo words."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2509_20563_b200 as fz  # noqa: E402
from paper_2509_20563_b200.data import smooth_trig_host  # noqa: E402

SEQ = [((64, 64, 64), "speed", 1e-4), ((17, 19, 23), "default", 1e-4), ((64, 64, 64), "default", 1e-2),
       ((33, 31), "default", 1e-4), ((4096,), "default", 1e-4), ((64, 64, 64), "default", 1e-4),
       ((128, 96), "speed", 1e-2), ((32, 40, 48), "default", 1e-6), ((64, 64, 64), "speed", 1e-4),
       ((8, 9, 10), "speed", 1e-4), ((131072,), "speed", 1e-4), ((64, 64, 64), "quality", 1e-4),
       ((65, 65), "default", 1e-4), ((64, 64, 64), "default", 1e-2)]


@pytest.mark.parametrize("rounds", [3])
def test_interleaved_shapes_match_oracle(oracle, rounds):
    for r in range(rounds):
        for q, (dims, preset, rel) in enumerate(SEQ):
            x = smooth_trig_host(dims, 100 * r + q)
            a = fz.compress(fz.Field(dims, x), fz.ErrorBoundSpec(fz.ErrorMode.VALUE_RANGE_RELATIVE, rel), preset)
            blob = fz.serialize_archive(a)
            want = oracle.compress(x, dims, 1, rel, preset)
            assert blob == want, (r, dims, preset, rel)
            rec = fz.decompress(fz.parse_archive(blob))
            _, orec = oracle.decompress(want)
            assert rec.data.tobytes() == orec.tobytes(), (r, dims, preset, rel)
