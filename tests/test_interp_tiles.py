"""2D G-Interp through the shared-memory tile kernels (interp.cu run_tiles2d:
levels stride/2..4 on the 4-lattice, levels 2, 1 on the field, 64 x 64 tiles
with recomputed halos).  Reference: fzpipe predict.py:147-201 (the same
stencil, boundary rules and quantizer as the grid-wide passes).

Shapes straddle the tile edges (63/64/65, one-row/one-column remainders,
fields narrower than a halo) and both anchor strides (16 = quality, 8 = the
profiled pipeline's alternative).  Small cases: byte-exact archive and
reconstruction vs the oracle.  Large cases: the tile path and the grid-wide
pass path (FZB_INTERP_PASSES=1, read per call) must produce identical
archives and reconstructions, and the reconstruction honours the bound."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2509_20563_b200 as fz  # noqa: E402
from paper_2509_20563_b200.data import noise_host, smooth_trig_host  # noqa: E402

SMALL = [(2, 2), (2, 300), (300, 2), (3, 5), (17, 18), (63, 64), (64, 64), (65, 65), (64, 129), (129, 63),
         (70, 75), (100, 37), (200, 300)]


def _x(dims, kind, seed):
    return noise_host(int(np.prod(dims)), seed).reshape(dims) if kind == "noise" else smooth_trig_host(dims, seed)


def _eb(rel):
    return fz.ErrorBoundSpec(fz.ErrorMode.VALUE_RANGE_RELATIVE, rel)


@pytest.mark.parametrize("dims", SMALL)
@pytest.mark.parametrize("kind,rel", [("trig", 1e-4), ("noise", 1e-2), ("trig", 1e-7)])
def test_tiles_bit_exact_vs_oracle(oracle, dims, kind, rel):
    x = _x(dims, kind, 11)
    a = fz.compress(fz.Field(dims, x), _eb(rel), "quality")
    blob = fz.serialize_archive(a)
    want = oracle.compress(x.ravel(), dims, 1, rel, "quality")
    assert blob == want
    _, orec = oracle.decompress(want)
    assert fz.decompress(fz.parse_archive(blob)).data.tobytes() == orec.tobytes()


@pytest.mark.parametrize("dims", [(64, 64), (65, 130), (200, 300)])
def test_tiles_profiled_stride8_vs_oracle(oracle, dims):
    # noise at 1e-3 prefers stride 8 / linear in the profile for some shapes;
    # both choices go through run_tiles2d (coarse kernel htop 1 or 2)
    for kind, rel in [("noise", 1e-3), ("trig", 1e-4)]:
        x = _x(dims, kind, 3)
        blob = fz.serialize_archive(fz.compress(fz.Field(dims, x), _eb(rel), "q-profiled"))
        want = oracle.compress(x.ravel(), dims, 1, rel, "q-profiled")
        assert blob == want
        _, orec = oracle.decompress(want)
        assert fz.decompress(fz.parse_archive(blob)).data.tobytes() == orec.tobytes()


@pytest.mark.parametrize("dims", [(1800, 3600), (1001, 2049), (4097, 65)])
def test_tiles_equal_grid_passes_large(dims, monkeypatch):
    x = smooth_trig_host(dims, 7)
    out = {}
    for mode in ("tiles", "passes"):
        if mode == "passes":
            monkeypatch.setenv("FZB_INTERP_PASSES", "1")
        blob = fz.serialize_archive(fz.compress(fz.Field(dims, x), _eb(1e-4), "quality"))
        rec = fz.decompress(fz.parse_archive(blob)).data
        out[mode] = (blob, rec.tobytes())
        monkeypatch.delenv("FZB_INTERP_PASSES", raising=False)
    assert out["tiles"][0] == out["passes"][0]
    assert out["tiles"][1] == out["passes"][1]
    rec = np.frombuffer(out["tiles"][1], dtype=np.float32)
    eb = 1e-4 * (float(x.max()) - float(x.min()))
    assert np.abs(rec.astype(np.float64) - x.ravel().astype(np.float64)).max() <= eb
    assert os.environ.get("FZB_INTERP_PASSES") is None
