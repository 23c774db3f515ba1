"""GPU parity: the sm_100a path against the reference (golden fixtures made
by fzpipe) and against the C oracle on larger seeded inputs.  Integer and
byte outputs must be bit-exact; reconstructions bitwise equal to the
reference's (0 ulp) and within the error bound."""

import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2509_20563_b200 as fz  # noqa: E402
from paper_2509_20563_b200 import encode as enc, errors as E, predict as pr  # noqa: E402
from paper_2509_20563_b200.core import ErrorBoundSpec, ErrorMode, Field, ResolvedBound  # noqa: E402

PRED = np.load(os.path.join(GOLDEN, "predict.npz"))
ARCH = np.load(os.path.join(GOLDEN, "archives.npz"))
BOOKS = np.load(os.path.join(GOLDEN, "codebooks.npz"))
REL, ABS = ErrorMode.VALUE_RANGE_RELATIVE, ErrorMode.ABSOLUTE


def _case(name):
    g = lambda k: PRED[f"{name}__{k}"]
    f = Field(tuple(int(d) for d in g("dims")), g("orig"))
    eb = float(g("eb")[0])
    return g, f, ResolvedBound(eb, float(f.data.min()), float(f.data.max())), int(g("radius")[0])


# ---------------------------------------------------------------- predictors

@pytest.mark.parametrize("name", list(PRED["names"]))
def test_lorenzo_bit_exact_vs_reference(name):
    g, f, b, r = _case(name)
    q = pr.lorenzo_quantize(f, b, r)
    assert np.array_equal(q.codes, g("lz_codes"))
    assert np.array_equal(q.outlier_indices, g("lz_oidx"))
    assert q.outlier_values.tobytes() == g("lz_oval").tobytes()
    rec = pr.lorenzo_reconstruct(q, b)
    assert rec.data.tobytes() == g("lz_recon").tobytes()


@pytest.mark.parametrize("name", [n for n in PRED["names"] if f"{n}__ip_codes" in PRED])
def test_interp_bit_exact_vs_reference(name):
    g, f, b, r = _case(name)
    q, anchors = pr.interp_quantize(f, b, r)
    assert anchors == g("ip_anchors").tobytes()
    assert np.array_equal(q.codes, g("ip_codes"))
    assert np.array_equal(q.outlier_indices, g("ip_oidx"))
    rec = pr.interp_reconstruct(q, anchors, b)
    assert rec.data.tobytes() == g("ip_recon").tobytes()


@pytest.mark.parametrize("dims,eb,seed", [((48, 96, 130), 1e-4, 1), ((9, 33, 257), 1e-3, 2), ((3, 70, 90), 1e-4, 3),
                                          ((700, 333), 1e-4, 4), ((64, 2000), 1e-3, 5), ((2, 5, 3000), 1e-4, 6)])
def test_lorenzo_vs_oracle_multitile(oracle, dims, eb, seed):
    from paper_2509_20563_b200.data import smooth_trig_host
    x = smooth_trig_host(dims, seed)
    lo, hi = float(x.min()), float(x.max())
    e = eb * (hi - lo)
    codes, idx, vals, recon = oracle.lorenzo_quantize(x, dims, e)
    f = Field(dims, x)
    q = pr.lorenzo_quantize(f, ResolvedBound(e, lo, hi))
    assert np.array_equal(q.codes, codes)
    assert np.array_equal(q.outlier_indices, idx)
    assert pr.lorenzo_reconstruct(q, ResolvedBound(e, lo, hi)).data.tobytes() == recon.tobytes()


@pytest.mark.parametrize("n,kind,eb", [(2_000_000, "particle", 1e-4), (300_000, "particle", 1e-2),
                                       (40_000, "noise", 1e-4), (100_003, "trig", 1e-3)])
def test_lorenzo_1d_vs_oracle(oracle, n, kind, eb):
    from paper_2509_20563_b200 import data
    x = {"particle": lambda: data.particle1d_host(n, 1), "noise": lambda: data.noise_host(n, 2),
         "trig": lambda: data.smooth_trig_host((n,), 3)}[kind]()
    lo, hi = float(x.min()), float(x.max())
    e = eb * (hi - lo)
    codes, idx, vals, recon = oracle.lorenzo_quantize(x, (n,), e)
    q = pr.lorenzo_quantize(Field((n,), x), ResolvedBound(e, lo, hi))
    assert np.array_equal(q.codes, codes)
    assert np.array_equal(q.outlier_indices, idx)
    assert pr.lorenzo_reconstruct(q, ResolvedBound(e, lo, hi)).data.tobytes() == recon.tobytes()


def test_interp_vs_oracle_3d(oracle):
    from paper_2509_20563_b200.data import smooth_trig_host
    dims = (50, 67, 90)
    x = smooth_trig_host(dims, 8)
    lo, hi = float(x.min()), float(x.max())
    e = 1e-4 * (hi - lo)
    codes, idx, vals, recon, anchors = oracle.interp_quantize(x, dims, e)
    q, a = pr.interp_quantize(Field(dims, x), ResolvedBound(e, lo, hi))
    assert a == anchors and np.array_equal(q.codes, codes) and np.array_equal(q.outlier_indices, idx)
    assert pr.interp_reconstruct(q, a, ResolvedBound(e, lo, hi)).data.tobytes() == recon.tobytes()


# -------------------------------------------------------------------- codecs

def test_package_merge_matches_reference_codebooks():
    off = 0
    for nsym in BOOKS["sizes"]:
        h = BOOKS["hist"][off:off + nsym]
        want = BOOKS["lengths"][off:off + nsym]
        total = int(h.sum())
        cb = enc.build_codebook(enc.Histogram(h, total))
        assert np.array_equal(cb.code_lengths, want), nsym
        off += nsym


@pytest.mark.parametrize("seed", range(4))
def test_huffman_and_bitshuffle_bytes_vs_oracle(oracle, seed):
    rng = np.random.default_rng(seed)
    n = [1, 255, 4097, 300_001][seed]
    codes = np.clip(np.round(rng.normal(512, [1, 3, 20, 200][seed], n)), 0, 1023).astype(np.uint32)
    h = enc.histogram_exact(codes, 512)
    assert np.array_equal(h.bins, oracle.histogram(codes, 512))
    assert enc.histogram_topk(codes, 512) == h
    cb, stream, bits = enc.huffman_encode(codes, h)
    cl, ostream, obits = oracle.huffman_encode(codes, h.bins)
    assert np.array_equal(cb.code_lengths, cl) and bits == obits and stream == ostream
    assert np.array_equal(enc.huffman_decode(cb, stream, n), codes)
    assert np.array_equal(cb.canonical_codewords(), oracle.codewords(cl))
    bm, pay = enc.bitshuffle_encode(codes, 512)
    obm, opay = oracle.bitshuffle_encode(codes, 512)
    assert bm == obm and pay == opay
    assert np.array_equal(enc.bitshuffle_decode(bm, pay, n, 512), codes)


def test_reference_kats():
    # test_encode.py:118-138, 220-227 of the reference suite
    codes = np.full(100, 7, np.uint32)
    cb, stream, bits = enc.huffman_encode(codes, enc.histogram_exact(codes, 8))
    assert bits == 100 and len(stream) == 13 and cb.code_lengths[7] == 1 and cb.used_symbols == 1
    assert np.array_equal(enc.huffman_decode(cb, stream, 100), codes)
    codes = np.concatenate([np.full(c, s, np.uint32) for s, c in enumerate([4, 2, 1, 1])])
    cb, stream, bits = enc.huffman_encode(codes, enc.histogram_exact(codes, 2))
    assert bits == 14 and np.array_equal(enc.huffman_decode(cb, stream, codes.size), codes)
    bm, pay = enc.bitshuffle_encode(np.ones(256, np.uint32), 512)
    assert np.frombuffer(pay, "<u4").tolist() == [0xFFFFFFFF] * 8


def test_huffman_decode_error_classes_match_oracle(oracle):
    rng = np.random.default_rng(7)
    codes = np.clip(np.round(rng.normal(512, 4, 20000)), 0, 1023).astype(np.uint32)
    cb, stream, bits = enc.huffman_encode(codes, enc.histogram_exact(codes, 512))
    cases = [stream[:-1], stream + b"\x00", stream[:len(stream) // 2]]
    if bits & 7:
        cases.append(stream[:-1] + bytes([stream[-1] | 1]))
    for k in range(0, 8 * len(stream), max(1, 8 * len(stream) // 40)):  # single-bit flips
        s = bytearray(stream)
        s[k >> 3] ^= 1 << (7 - (k & 7))
        cases.append(bytes(s))
    for s in cases:
        try:
            want = oracle.huffman_decode(cb.code_lengths, s, codes.size)
            got = enc.huffman_decode(cb, s, codes.size)
            assert np.array_equal(got, want)
        except oracle.OracleError as e:
            with pytest.raises(getattr(E, e.kind)):
                enc.huffman_decode(cb, s, codes.size)


def test_bitshuffle_decode_errors():
    codes = np.full(300, 513, np.uint32)
    bm, pay = enc.bitshuffle_encode(codes, 512)
    with pytest.raises(E.Truncated):
        enc.bitshuffle_decode(bm[:-1], pay, 300, 512)
    with pytest.raises(E.BitmapPayloadMismatch):
        enc.bitshuffle_decode(bm + b"\x00", pay, 300, 512)
    with pytest.raises(E.BitmapPayloadMismatch):
        enc.bitshuffle_decode(bm, pay[:-4], 300, 512)
    with pytest.raises(E.CorruptPayload):  # 513 codes decoded with radius 256 -> code >= 2R
        enc.bitshuffle_decode(bm, pay, 300, 256)


# ------------------------------------------------------------------ pipeline

@pytest.mark.parametrize("name", list(ARCH["names"]))
@pytest.mark.parametrize("preset", ["default", "speed", "quality"])
def test_archives_byte_identical_to_reference(name, preset):
    g = lambda k: ARCH[f"{name}__{k}"]
    dims = tuple(int(d) for d in g("dims"))
    f = Field(dims, g("orig"))
    a = fz.compress(f, ErrorBoundSpec(ErrorMode(int(g("mode")[0])), float(g("mag")[0])), preset)
    blob = fz.serialize_archive(a)
    assert blob == g(f"{preset}__archive").tobytes()
    rec = fz.decompress(fz.parse_archive(blob))
    assert rec.data.tobytes() == g(f"{preset}__recon").tobytes()


def test_decompress_rejects_corruption_like_reference():
    blob = ARCH["smooth2d__default__archive"].tobytes()
    a = fz.parse_archive(blob)
    segs = list(a.segments)
    k, stream = segs[3]
    segs[3] = (k, stream + b"\x00")
    bad = fz.Archive(a.pipeline_id, a.eb_mode, a.eb_magnitude, a.data_min, a.data_max, a.dims, a.radius, tuple(segs))
    with pytest.raises(E.StageError) as ei:
        fz.decompress(bad)
    assert isinstance(ei.value.cause, E.CorruptStream)
    segs = list(a.segments)
    segs[0] = (segs[0][0], np.array([10 ** 9], "<u8").tobytes())
    segs[1] = (segs[1][0], np.array([1.0], "<f4").tobytes())
    bad = fz.Archive(a.pipeline_id, a.eb_mode, a.eb_magnitude, a.data_min, a.data_max, a.dims, a.radius, tuple(segs))
    with pytest.raises(E.StageError):
        fz.decompress(bad)


@pytest.mark.parametrize("preset", ["default", "speed", "quality"])
def test_full_size_c1_archive_matches_oracle(oracle, preset):
    """BASELINE config C1 (100x500x500 smooth_trig, rel 1e-4) at full size."""
    from paper_2509_20563_b200 import data
    dims = (100, 500, 500)
    x = data.smooth_trig_device(dims, 0).cpu().numpy()
    want = oracle.compress(x, dims, 1, 1e-4, preset)
    a = fz.compress(Field(dims, x), ErrorBoundSpec(REL, 1e-4), preset)
    assert fz.serialize_archive(a) == want
    rec = fz.decompress(a)
    _, orec = oracle.decompress(want)
    assert rec.data.tobytes() == orec.tobytes()
    assert float(np.max(np.abs(rec.data.astype(np.float64) - x))) <= a.resolved_bound().eb_abs


def test_lorenzo_1d_negative_zero_and_outliers(oracle):
    # -0.0 outliers followed by zero-code runs: recon must normalise to +0.0 exactly like the reference
    x = np.zeros(5000, np.float32)
    x[::7] = -0.0
    x[100] = 1e6
    x[101:400] = -0.0
    x[1000:1100] = np.linspace(-1, 1, 100, dtype=np.float32)
    e = 1e-3
    codes, idx, vals, recon = oracle.lorenzo_quantize(x, (x.size,), e, 4)
    lo, hi = float(x.min()), float(x.max())
    q = pr.lorenzo_quantize(Field((x.size,), x), ResolvedBound(e, lo, hi), 4)
    assert np.array_equal(q.codes, codes) and np.array_equal(q.outlier_indices, idx)
    assert pr.lorenzo_reconstruct(q, ResolvedBound(e, lo, hi)).data.tobytes() == recon.tobytes()


@pytest.mark.parametrize("preset", ["default", "speed"])
def test_full_size_c4_archive_matches_oracle(oracle, preset):
    """BASELINE config C4: HACC-shaped 1D particle field, 280,953,867 values, rel 1e-4."""
    from paper_2509_20563_b200 import data
    n = 280_953_867
    x = data.particle1d_device(n, 0).cpu().numpy()
    want = oracle.compress(x, (n,), 1, 1e-4, preset)
    a = fz.compress(Field((n,), x), ErrorBoundSpec(REL, 1e-4), preset)
    assert fz.serialize_archive(a) == want
    rec = fz.decompress(a)
    _, orec = oracle.decompress(want)
    assert rec.data.tobytes() == orec.tobytes()


@pytest.mark.parametrize("preset", ["default", "speed", "quality"])
def test_wire_block_is_the_serialized_archive(preset):
    # the device path lays the archive out serialized in one pinned block:
    # archive_buffer must equal the reference serialization byte for byte and
    # parse back (zero-copy) to an equal archive that decompresses identically
    import paper_2509_20563_b200 as fz
    from paper_2509_20563_b200.core import header_bytes
    dims = (40, 48, 64)
    from paper_2509_20563_b200.data import smooth_trig_host
    f = fz.Field(dims, smooth_trig_host(dims, 3))
    eb = fz.ErrorBoundSpec(fz.ErrorMode.VALUE_RANGE_RELATIVE, 1e-4)
    a = fz.compress(f, eb, preset)
    buf = fz.archive_buffer(a)
    ref = header_bytes(a) + b"".join(bytes(p) for _, p in a.segments)
    assert bytes(buf) == ref == fz.serialize_archive(a)
    b = fz.parse_archive(buf)
    assert b == a
    assert fz.decompress(b).data.tobytes() == fz.decompress(a).data.tobytes()


@pytest.mark.parametrize("preset,dims", [("default", (40, 48, 64)), ("speed", (33, 40, 64)), ("quality", (96, 160)),
                                         ("default", (20_000,))])
def test_cuda_graph_round_trip(preset, dims):
    # the captured device DAG replays on new input data (static input
    # tensor) and yields the eager path's archive and reconstruction
    import torch
    from paper_2509_20563_b200.data import smooth_trig_host
    from paper_2509_20563_b200.device import graph_engine, pad3
    from paper_2509_20563_b200.pipeline import get_pipeline
    eng = graph_engine()
    spec = get_pipeline(preset)
    kw = dict(pipeline_id=spec.id, predictor=spec.predictor, codec=spec.primary_codec, radius=spec.radius())
    n = int(np.prod(dims))
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    eb = fz.ErrorBoundSpec(fz.ErrorMode.VALUE_RANGE_RELATIVE, 1e-4)
    for seed in range(3):
        host = smooth_trig_host(dims, seed)
        with torch.cuda.stream(eng.stream):
            x.copy_(torch.from_numpy(host))
        da = eng.compress_graphed(x, dims, 1, 1e-4, **kw)
        lo, hi, segs, _ = eng.finish(da)
        ref = fz.compress(fz.Field(dims, host), eb, preset)
        assert [(k, bytes(p)) for k, p in segs] == [(k, bytes(p)) for k, p in ref.segments]
        sz = eng.sizes(da)
        eng.decompress_graphed(da, sz, 1e-4 * (sz["hi"] - sz["lo"]), out)
        eng._sync()
        assert out.cpu().numpy().tobytes() == fz.decompress(ref).data.tobytes()


@pytest.mark.parametrize("preset", ["default", "speed", "quality"])
def test_graph_variants_bytes_equal_sequential(preset):
    # pipeline.py:650-660 / 583-591 graph variants: bytewise identical to the
    # sequential calls (test_pipeline.py:281-297); here they replay CUDA graphs
    from paper_2509_20563_b200.data import smooth_trig_host
    dims = (48, 40, 64)
    eb = fz.ErrorBoundSpec(fz.ErrorMode.VALUE_RANGE_RELATIVE, 1e-4)
    for seed in range(2):
        f = fz.Field(dims, smooth_trig_host(dims, seed))
        a = fz.compress_via_graph(f, eb, preset)
        assert fz.serialize_archive(a) == fz.serialize_archive(fz.compress(f, eb, preset))
        assert fz.decompress_via_graph(a).data.tobytes() == fz.decompress(a).data.tobytes()


# ------------------------------------------------------------------ edge cases

EDGE_DIMS = [(1,), (2,), (7,), (33,), (1, 1, 1), (1, 1, 5), (2, 2, 2), (3, 3), (1, 64), (64, 1), (17, 17),
             (4, 5, 6), (16, 17, 18), (1, 2, 3), (5, 1, 9)]


@pytest.mark.parametrize("dims", EDGE_DIMS)
@pytest.mark.parametrize("preset", ["default", "speed", "quality"])
def test_tiny_and_ragged_fields_match_oracle(oracle, dims, preset):
    # tiny / degenerate extents: every kernel's partial-tile, partial-block and
    # single-element paths (and the interp -> Lorenzo fallback) vs the oracle
    rng = np.random.default_rng(sum(dims) + len(preset))
    x = (np.cumsum(rng.normal(0, 1, int(np.prod(dims)))) * 0.1).astype(np.float32)
    want = oracle.compress(x, dims, 1, 1e-3, preset)
    a = fz.compress(Field(dims, x), ErrorBoundSpec(REL, 1e-3), preset)
    assert fz.serialize_archive(a) == want
    rec = fz.decompress(a)
    _, orec = oracle.decompress(want)
    assert rec.data.tobytes() == orec.tobytes()


@pytest.mark.parametrize("preset", ["default", "speed", "quality"])
@pytest.mark.parametrize("case", ["constant", "abs_tiny_eb", "abs_huge_eb", "two_values"])
def test_bound_edge_cases_match_oracle(oracle, preset, case):
    # constant field (header-only archive), an absolute bound so small that
    # almost everything is an outlier, one so large that every code is zero,
    # and a two-valued field
    dims = (24, 40, 36)
    n = int(np.prod(dims))
    x = np.sin(np.arange(n, dtype=np.float64) * 0.01).astype(np.float32)
    mode, mag = 1, 1e-3
    if case == "constant":
        x = np.full(n, 3.25, np.float32)
    elif case == "abs_tiny_eb":
        mode, mag = 0, 1e-9
    elif case == "abs_huge_eb":
        mode, mag = 0, 10.0
    else:
        x = np.where(np.arange(n) % 3 == 0, -1.5, 2.0).astype(np.float32)
    want = oracle.compress(x, dims, mode, mag, preset)
    eb = ErrorBoundSpec(ABS if mode == 0 else REL, mag)
    a = fz.compress(Field(dims, x), eb, preset)
    assert fz.serialize_archive(a) == want
    rec = fz.decompress(a)
    _, orec = oracle.decompress(want)
    assert rec.data.tobytes() == orec.tobytes()
