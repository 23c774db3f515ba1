"""Opt-in dual-quant Lorenzo pipelines (ids 3 'dq-speed' = dual-quant +
bitshuffle, 4 'dq-default' = dual-quant + Huffman; north_star items 1 and 4).
They have no reference counterpart (they change the reference's codes by
design), so their oracle is oracle.fzoracle.dq_* -- a
numpy statement of the spec in csrc/dualquant.cu.  CPU: the spec's own
properties.  GPU: archives and reconstructions bit-exact vs that oracle,
error bound, the range error."""

import numpy as np
import pytest

from paper_2509_20563_b200.data import noise_host, particle1d_host, smooth_trig_host

SHAPES = [(1000,), (50000,), ((1 << 20) + 7,), (50, 70), (333, 129), (20, 30, 40), (17, 19, 23), (64, 64, 64)]


def _field(dims, seed, kind="trig"):
    if kind == "noise":
        return noise_host(int(np.prod(dims)), seed)
    if len(dims) == 1 and kind == "particle":
        return particle1d_host(dims[0], seed)
    return smooth_trig_host(dims, seed)


@pytest.mark.parametrize("dims", SHAPES[:6])
@pytest.mark.parametrize("rel", [1e-2, 1e-4])
def test_oracle_dualquant_round_trip_within_bound(oracle, dims, rel):
    x = _field(dims, 1)
    for p in ("dq-speed", "dq-default"):
        blob = oracle.compress(x, dims, 1, rel, p)
        _, r = oracle.decompress(blob)
        eb = rel * (float(x.max()) - float(x.min()))
        assert np.abs(r.astype(np.float64) - x.astype(np.float64)).max() <= eb


def test_oracle_dualquant_spec_properties(oracle):
    # a linear ramp in 1D: every delta after the first is the constant step
    x = (np.arange(1000, dtype=np.float64) * 0.25).astype(np.float32)
    codes, idx, vals, deltas = oracle.dq_quantize(x, (1000,), 0.125 / 2, 512)   # 2eb = 0.125 -> p = 2t
    assert set(codes[1:].tolist()) == {514} and idx.size == 0
    # a spike becomes outliers (delta >= R) with the exact value restored
    y = np.zeros((8, 9), np.float32)
    y[3, 4] = 1e4
    codes, idx, vals, deltas = oracle.dq_quantize(y.reshape(-1), (8, 9), 0.5, 512)
    assert 3 * 9 + 4 in idx.tolist()
    rec = oracle.dq_reconstruct(codes, idx, vals, deltas, (8, 9), 0.5, 512)
    assert rec.reshape(8, 9)[3, 4] == np.float32(1e4)


gpu = pytest.mark.gpu


def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2509_20563_b200 as fz
    return fz


@gpu
@pytest.mark.parametrize("dims", SHAPES)
@pytest.mark.parametrize("preset", ["dq-speed", "dq-default"])
@pytest.mark.parametrize("kind,rel", [("trig", 1e-3), ("trig", 1e-5), ("noise", 1e-5)])
def test_gpu_dualquant_bit_exact_vs_oracle(oracle, dims, preset, kind, rel):
    fz = _gpu()
    x = _field(dims, 7, kind)
    a = fz.compress(fz.Field(dims, x), fz.ErrorBoundSpec(fz.ErrorMode.VALUE_RANGE_RELATIVE, rel), preset)
    blob = fz.serialize_archive(a)
    want = oracle.compress(x, dims, 1, rel, preset)
    assert blob == want
    r = fz.decompress(fz.parse_archive(want))
    _, orec = oracle.decompress(want)
    assert r.data.tobytes() == orec.tobytes()
    eb = a.resolved_bound().eb_abs
    assert np.abs(r.data.astype(np.float64) - x.astype(np.float64)).max() <= eb


@gpu
def test_gpu_dualquant_range_error():
    fz = _gpu()
    x = smooth_trig_host((64, 64), 2) + np.float32(1000.0)
    with pytest.raises(Exception, match="2\\^27"):
        fz.compress(fz.Field((64, 64), x), fz.ErrorBoundSpec(fz.ErrorMode.VALUE_RANGE_RELATIVE, 1e-9), "dq-speed")
