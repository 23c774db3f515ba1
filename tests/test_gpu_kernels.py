"""GPU parity for the round-1 kernels (v7 Lorenzo wavefront, bitshuffle
transpose, Huffman multi-symbol decode, privatised histogram) against the C
oracle: shapes that hit partial tiles in i and j, every v7 tile
configuration, small radii (outlier-heavy), signed zeros and constant runs,
alphabets beyond the 12-bit LUT fast path, and sizes off every block
boundary.  Integer outputs bit-exact, reconstructions bitwise equal."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2509_20563_b200 import encode as enc, predict as pr  # noqa: E402
from paper_2509_20563_b200.core import Field, ResolvedBound  # noqa: E402
from paper_2509_20563_b200.data import smooth_trig_host  # noqa: E402


def _lorenzo_check(oracle, x, dims, e, radius=512):
    lo, hi = float(x.min()), float(x.max())
    codes, idx, vals, recon = oracle.lorenzo_quantize(x, dims, e, radius)
    b = ResolvedBound(e, lo, hi)
    q = pr.lorenzo_quantize(Field(dims, x), b, radius)
    assert np.array_equal(q.codes, codes)
    assert np.array_equal(q.outlier_indices, idx)
    assert q.outlier_values.tobytes() == vals.tobytes()
    assert pr.lorenzo_reconstruct(q, b).data.tobytes() == recon.tobytes()
    return int(idx.size)


# n2 % 4 == 0 throughout: these run the v7 wavefront (others fall back to v4)
V7_SHAPES = [(8, 32, 64), (9, 33, 64), (17, 65, 100), (48, 96, 132), (33, 40, 36), (100, 20, 8), (5, 130, 44)]


@pytest.mark.parametrize("dims", V7_SHAPES)
def test_v7_lorenzo_shapes(oracle, dims):
    x = smooth_trig_host(dims, sum(dims))
    _lorenzo_check(oracle, x, dims, 1e-4 * float(x.max() - x.min()))


@pytest.mark.parametrize("cfg", ["4x2", "2x2", "1x1", "1x2", "8x1", "4x1", "2x4", "8x2", "4x4", "4x3"])
def test_v7_tile_configs(oracle, cfg, monkeypatch):
    dims = (37, 70, 48)
    monkeypatch.setenv("FZB_LZ_CFG", cfg)
    x = smooth_trig_host(dims, 11)
    _lorenzo_check(oracle, x, dims, 1e-3 * float(x.max() - x.min()))


@pytest.mark.parametrize("radius", [1, 2, 8, 32768])
def test_v7_outlier_heavy(oracle, radius):
    dims = (20, 40, 52)
    x = smooth_trig_host(dims, 5)
    k = _lorenzo_check(oracle, x, dims, 1e-5 * float(x.max() - x.min()), radius)
    if radius <= 8:
        assert k > 0


def test_v7_signed_zeros_and_constant_runs(oracle):
    dims = (12, 40, 64)
    rng = np.random.default_rng(3)
    x = smooth_trig_host(dims, 2).reshape(dims)
    x[:, :, 10:30] = 0.0
    x[:, 5:9, :] = -0.0
    x[3] = 1.25
    x = x.reshape(-1).astype(np.float32)
    x[rng.integers(0, x.size, 200)] *= -1
    _lorenzo_check(oracle, x, dims, 1e-4 * float(x.max() - x.min()))


def test_v7_2d(oracle):
    dims = (130, 1000)
    x = smooth_trig_host(dims, 9)
    _lorenzo_check(oracle, x, dims, 1e-4 * float(x.max() - x.min()))


@pytest.mark.parametrize("n", [1, 7, 255, 256, 257, 8191, 8192, 8193, 100_003, 1 << 20])
def test_bitshuffle_sizes(oracle, n):
    rng = np.random.default_rng(n)
    codes = np.clip(np.round(rng.normal(512, 3, n)), 0, 1023).astype(np.uint32)
    codes[rng.integers(0, n, max(1, n // 50))] = rng.integers(0, 1024, max(1, n // 50))
    bm, pay = enc.bitshuffle_encode(codes, 512)
    obm, opay = oracle.bitshuffle_encode(codes, 512)
    assert bm == obm and pay == opay
    assert np.array_equal(enc.bitshuffle_decode(bm, pay, n, 512), codes)


@pytest.mark.parametrize("radius,spread", [(512, 1.0), (512, 60.0), (2048, 300.0), (4096, 900.0)])
def test_huffman_alphabets(oracle, radius, spread):
    # radius 4096 -> 8192 symbols: the 12-bit LUT holds one symbol per window
    rng = np.random.default_rng(int(spread))
    n = 200_001
    codes = np.clip(np.round(rng.normal(radius, spread, n)), 0, 2 * radius - 1).astype(np.uint32)
    h = enc.histogram_exact(codes, radius)
    assert np.array_equal(h.bins, oracle.histogram(codes, radius))
    cb, stream, bits = enc.huffman_encode(codes, h)
    cl, ostream, obits = oracle.huffman_encode(codes, h.bins)
    assert np.array_equal(cb.code_lengths, cl) and bits == obits and stream == ostream
    assert np.array_equal(enc.huffman_decode(cb, stream, n), codes)


def test_histogram_runs_and_tail(oracle):
    n = 1_000_003   # not a multiple of 8
    codes = np.full(n, 512, np.uint32)
    codes[::97] = 3
    codes[-5:] = 1023
    h = enc.histogram_exact(codes, 512)
    assert np.array_equal(h.bins, oracle.histogram(codes, 512))


# ------------------------------------------------------------------ batches

@pytest.mark.parametrize("preset,dims", [("speed", (24, 40, 64)), ("default", (17, 65, 64)), ("default", (96, 128))])
def test_batch_archives_identical(preset, dims):
    import paper_2509_20563_b200 as fz
    eb = fz.ErrorBoundSpec(fz.ErrorMode.VALUE_RANGE_RELATIVE, 1e-4)
    fields = [fz.Field(dims, smooth_trig_host(dims, s)) for s in range(3)]
    single = [fz.serialize_archive(fz.compress(f, eb, preset)) for f in fields]
    batch = fz.compress_batch(fields, eb, preset)
    assert [fz.serialize_archive(a) for a in batch] == single
    parsed = [fz.parse_archive(b) for b in single]
    recs = fz.decompress_batch(parsed)
    for a, r in zip(parsed, recs):
        assert r.data.tobytes() == fz.decompress(a).data.tobytes()


# ------------------------------------------------------------------ quality

@pytest.mark.parametrize("n", [1, 7, 8, 129, 1000, 100_003, 1 << 20, 3_000_017])
def test_quality_device_bit_identical(n):
    from paper_2509_20563_b200 import metrics
    rng = np.random.default_rng(n)
    o = (rng.normal(0, 1, n) * 3).astype(np.float32)
    r = (o + rng.uniform(-1e-3, 1e-3, n)).astype(np.float32)
    r[::7] = o[::7]   # some exact elements
    host = metrics.quality_arrays(o, r, 1e-3)
    dev = metrics.quality_device(torch.from_numpy(o).cuda(), torch.from_numpy(r).cuda(), (n,), 1e-3)
    assert dev == host   # every field equal (floats compared exactly)


def test_quality_device_edge_cases():
    from paper_2509_20563_b200 import metrics
    z = np.zeros(1000, np.float32)
    z[::3] = -0.0
    for o, r in [(z, z.copy()), (z, z + np.float32(1e-3)), (np.linspace(-1, 1, 999, dtype=np.float32),) * 2]:
        host = metrics.quality_arrays(o, r, None)
        dev = metrics.quality_device(torch.from_numpy(o).cuda(), torch.from_numpy(np.ascontiguousarray(r)).cuda(),
                                     (o.size,), None)
        assert dev == host


@pytest.mark.parametrize("seed", range(12))
def test_huffman_build_ties_vs_oracle(oracle, seed):
    # tie-heavy histograms (many equal small counts, 2..300 used symbols) drive
    # both build paths (single-warp <= 256 used symbols, block otherwise) and
    # package lists that are not sorted by (weight, tiebreak); the stream
    # checks the device-built canonical codewords too
    rng = np.random.default_rng(seed)
    m = int(rng.integers(2, 300))
    used = rng.choice(1024, m, replace=False)
    kind = seed % 3
    reps = (rng.integers(1, 4, m) if kind == 0 else
            2 ** rng.integers(0, 12, m) if kind == 1 else rng.geometric(0.05, m))
    codes = rng.permutation(np.repeat(used, reps)).astype(np.uint32)
    h = enc.histogram_exact(codes, 512)
    cb, stream, bits = enc.huffman_encode(codes, h)
    cl, ostream, obits = oracle.huffman_encode(codes, h.bins)
    assert np.array_equal(cb.code_lengths, cl) and bits == obits and stream == ostream
    assert np.array_equal(enc.huffman_decode(cb, stream, codes.size), codes)


@pytest.mark.parametrize("seed", range(15))
def test_huffman_build_large_alphabets_vs_oracle(oracle, seed):
    # 257..3000 used symbols: the whole-CTA rank-search merge (shared memory,
    # up to 2048 symbols, including its fixed-point exit) and the global-
    # memory path beyond; tie-heavy, power-of-two and geometric weights
    rng = np.random.default_rng(100 + seed)
    radius = (512, 1024, 2048)[seed % 3]
    m = int(rng.integers(257, min(2 * radius, 3000)))
    used = rng.choice(2 * radius, m, replace=False)
    kind = (seed // 3) % 3
    reps = (rng.integers(1, 4, m) if kind == 0 else
            2 ** rng.integers(0, 10, m) if kind == 1 else rng.geometric(0.02, m))
    codes = rng.permutation(np.repeat(used, reps)).astype(np.uint32)
    h = enc.histogram_exact(codes, radius)
    cb, stream, bits = enc.huffman_encode(codes, h)
    cl, ostream, obits = oracle.huffman_encode(codes, h.bins)
    assert np.array_equal(cb.code_lengths, cl) and bits == obits and stream == ostream
    assert np.array_equal(enc.huffman_decode(cb, stream, codes.size), codes)


@pytest.mark.parametrize("n,seed", [(4096 * 5, 0), (4096 * 5 + 3, 1), (4096 * 7 + 4095, 2), (12345, 3), (8191, 4),
                                    (4096 * 64, 5), (4096 * 64 + 8, 6)])
def test_histogram_chunk_flags_and_flagged_encode(oracle, n, seed):
    # fzb_histogram_chunks flags exactly the 4096-code chunks holding a code
    # != R (incl. a chunk's first/last code and the partial tail), and the
    # flag-driven count pass (fzb_huffman_encode_chunks) writes the same
    # stream as the unflagged one and the oracle
    from paper_2509_20563_b200.encode import _build, _fetch, _status, _upload_codes
    from paper_2509_20563_b200.device import _p, default_engine
    rng = np.random.default_rng(seed)
    radius = 512
    R = radius
    c = np.full(n, R, np.uint16)
    pos = list(rng.choice(n, min(n, 40), replace=False)) + [0, n - 1, min(n - 1, 4095), min(n - 1, 4096)]
    c[pos] = rng.integers(R - 20, R + 20, len(pos)).astype(np.uint16)
    c[min(n - 1, 8192 + 7)] = R   # may undo one of the above: flags must follow the final bytes
    eng = default_engine()
    nsym = 2 * radius
    d = _upload_codes(eng, "t_codes", c)
    bins = eng.buf("t_bins", 8 * nsym)
    nc = (n + 4095) // 4096
    notr = eng.buf("t_notr", nc)
    st = eng.buf("dstatus", 8, zero=True)
    eng._call("fzb_histogram_chunks", _p(d), n, nsym, _p(bins), _p(notr), _p(st), eng.sp)
    got_bins = np.frombuffer(_fetch(eng, bins, 8 * nsym), np.uint64)
    assert np.array_equal(got_bins, np.bincount(c, minlength=nsym).astype(np.uint64))
    got_flags = np.frombuffer(_fetch(eng, notr, nc), np.uint8)
    want_flags = np.array([np.any(c[4096 * k:4096 * (k + 1)] != R) for k in range(nc)], np.uint8)
    assert np.array_equal(got_flags, want_flags)
    lengths, cw, bc = _build(eng, got_bins.copy())
    cap = 4 * n + 16
    streams = []
    for flagged in (False, True):
        out = eng.buf(f"t_out{int(flagged)}", cap, zero=True)
        ws = eng.buf("t_ws", eng.lib.fzb_huffman_encode_workspace_bytes(n))
        if flagged:
            eng._call("fzb_huffman_encode_chunks", _p(d), n, _p(lengths), _p(cw), nsym, _p(bc), _p(notr), _p(out), cap,
                      _p(ws), ws.numel(), _p(st), eng.sp)
        else:
            eng._call("fzb_huffman_encode", _p(d), n, _p(lengths), _p(cw), nsym, _p(bc), _p(out), cap, _p(ws),
                      ws.numel(), _p(st), eng.sp)
        bits = int(np.frombuffer(_fetch(eng, bc, 8), np.uint64)[0])
        streams.append(_fetch(eng, out, (bits + 7) // 8))
    assert _status(eng) == 0
    assert streams[0] == streams[1]
    _, ostream, _ = oracle.huffman_encode(c.astype(np.uint32), got_bins.copy())
    assert streams[1] == ostream


@pytest.mark.parametrize("n,seed", [(4096 * 3 + 5, 0), (1000003, 1), (8 * 1024, 2), (4099, 3), (65536 + 1, 4)])
def test_huffman_low_entropy_prefill_path(oracle, n, seed):
    # a dominant zero code with the 1-bit codeword "0" at <= 1.125 bits per
    # symbol takes the decoder's s0 prefill + skip-all-s0-chunk path: other
    # symbols at 8-symbol chunk edges, at the ends, and n % 8 != 0
    rng = np.random.default_rng(seed)
    radius = 512
    c = np.full(n, radius, np.uint32)
    k = max(1, n // 200)
    pos = np.unique(np.concatenate([rng.choice(n, k, replace=False), [0, n - 1],
                                    np.arange(7, n, 4096)[:8], np.arange(8, n, 4096)[:8]]))
    c[pos] = rng.integers(radius - 3, radius + 4, pos.size)
    h = enc.histogram_exact(c, radius)
    cb, stream, bits = enc.huffman_encode(c, h)
    assert bits * 8 <= 9 * n                       # the prefill regime
    assert cb.code_lengths[radius] == 1            # R has a 1-bit codeword
    cl, ostream, obits = oracle.huffman_encode(c, h.bins)
    assert np.array_equal(cb.code_lengths, cl) and stream == ostream
    assert np.array_equal(enc.huffman_decode(cb, stream, n), c)
