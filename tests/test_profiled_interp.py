"""Opt-in pipeline 5 'q-profiled': G-Interp whose anchor stride (16 | 8) and
interpolation weights (cubic | linear | natural cubic) are chosen per field by
sampled profiling (cuSZ-i / QoZ; north_star item 2).  No reference
counterpart; the oracle's interp_profile is the numpy statement of the
kernel's integer cost, so the choice and the archive must be bit-exact."""

import numpy as np
import pytest

from paper_2509_20563_b200.data import noise_host, smooth_trig_host

CASES = [((50, 70, 90), "trig", 1e-4), ((1800, 360), "trig", 1e-4), ((64, 64, 64), "noise", 1e-3),
         ((40, 200), "noise", 1e-2), ((33, 17, 65), "trig", 1e-3), ((17, 18), "trig", 1e-2)]


def _x(dims, kind, seed=5):
    return noise_host(int(np.prod(dims)), seed) if kind == "noise" else smooth_trig_host(dims, seed)


@pytest.mark.parametrize("dims,kind,rel", CASES)
def test_oracle_profiled_round_trip(oracle, dims, kind, rel):
    x = _x(dims, kind)
    blob = oracle.compress(x, dims, 1, rel, "q-profiled")
    _, r = oracle.decompress(blob)
    eb = rel * (float(x.max()) - float(x.min()))
    assert np.abs(r.astype(np.float64) - x.astype(np.float64)).max() <= eb


def test_oracle_profile_prefers_linear_on_noise(oracle):
    x = _x((64, 64, 64), "noise")
    sc = oracle.interp_profile(x, (64, 64, 64), 1e-3)
    stride, wi = oracle.profile_choice(sc)
    assert wi == 1 and stride == 16, (sc, stride, wi)
    y = _x((64, 64, 64), "trig")
    assert oracle.profile_choice(oracle.interp_profile(y, (64, 64, 64), 1e-4 * 4)) == (16, 0)


@pytest.mark.gpu
@pytest.mark.parametrize("dims,kind,rel", CASES)
def test_gpu_profiled_bit_exact_vs_oracle(oracle, dims, kind, rel):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2509_20563_b200 as fz
    x = _x(dims, kind)
    a = fz.compress(fz.Field(dims, x), fz.ErrorBoundSpec(fz.ErrorMode.VALUE_RANGE_RELATIVE, rel), "q-profiled")
    want = oracle.compress(x, dims, 1, rel, "q-profiled")
    assert fz.serialize_archive(a) == want
    r = fz.decompress(fz.parse_archive(want))
    _, orec = oracle.decompress(want)
    assert r.data.tobytes() == orec.tobytes()
