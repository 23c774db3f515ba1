"""Boundary fidelity on the GPU: the *_with_timing stage keys, the graph
variants (two-stream CUDA graphs, replayed with new archives), stage
attribution of errors, pickling of device-made archives, and the graph
cache's buffer lifetime (shape A, larger shape B, then A again)."""

import copy
import pickle

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2509_20563_b200 as fz  # noqa: E402
from paper_2509_20563_b200 import errors as E  # noqa: E402
from paper_2509_20563_b200.core import ErrorBoundSpec, ErrorMode, Field  # noqa: E402
from paper_2509_20563_b200.data import smooth_trig_host  # noqa: E402
from paper_2509_20563_b200.pipeline import PipelineSpec, StageKind, StageSpec, get_pipeline  # noqa: E402

REL = ErrorMode.VALUE_RANGE_RELATIVE
EB = ErrorBoundSpec(REL, 1e-4)


@pytest.mark.parametrize("preset", ["default", "speed", "quality"])
def test_compress_with_timing_keys_are_stage_names(preset):
    # pipeline.py:345-379: one entry per executed stage, keyed by its name
    f = Field((24, 40, 36), smooth_trig_host((24, 40, 36), 1))
    a, t = fz.compress_with_timing(f, EB, preset)
    spec = get_pipeline(preset)
    want = {s.name for s in spec.stages}
    assert set(t) == want
    assert all(isinstance(v, float) and v >= 0.0 for v in t.values())
    assert t[spec.stage_of(StageKind.PREDICT).name] > 0.0
    assert fz.serialize_archive(a) == fz.serialize_archive(fz.compress(f, EB, preset))


def test_compress_with_timing_constant_field_is_empty():
    # pipeline.py:360-363: a constant field returns before any stage runs
    f = Field((10, 10), np.full(100, 2.5, np.float32))
    a, t = fz.compress_with_timing(f, EB, "default")
    assert t == {} and a.segments == ()


@pytest.mark.parametrize("preset", ["default", "speed", "quality"])
def test_decompress_with_timing_keys(preset):
    # pipeline.py:439-466: unwrap, decode-codes, decode-outliers, reconstruct
    f = Field((24, 40, 36), smooth_trig_host((24, 40, 36), 2))
    a = fz.compress(f, EB, preset)
    r, t = fz.decompress_with_timing(a)
    assert set(t) == {"unwrap", "decode-codes", "decode-outliers", "reconstruct"}
    assert t["decode-codes"] > 0.0 and t["reconstruct"] > 0.0
    assert r.data.tobytes() == fz.decompress(a).data.tobytes()


def test_timing_keys_custom_stage_names_and_secondary():
    # a custom spec: preprocess + renamed stages + a secondary codec stage
    S, K = StageSpec, StageKind
    spec = PipelineSpec(77, (S("prep", K.PREPROCESS, {"op": "identity"}), S("lz", K.PREDICT, {"predictor": "lorenzo"}),
                             S("hist", K.ANALYSIS, {"method": "exact"}), S("hf", K.PRIMARY_CODEC, {"codec": "huffman"}),
                             S("rle", K.SECONDARY_CODEC, {"codec_id": "0"})))
    f = Field((16, 30, 20), smooth_trig_host((16, 30, 20), 3))
    a, t = fz.compress_with_timing(f, EB, spec)
    assert set(t) == {"prep", "lz", "hist", "hf", "rle"}
    r = fz.decompress(a, spec)
    assert r.data.tobytes() == fz.decompress(fz.compress(f, EB, "default")).data.tobytes()


@pytest.mark.parametrize("preset", ["default", "speed", "quality"])
def test_decompress_via_graph_replays_new_archives(preset):
    # the captured two-stream decompress graph is replayed for later archives
    # of the same shape and payload sizes (payloads restaged on the host);
    # every replay must equal the eager path bit for bit
    dims = (32, 48, 40)
    arcs = [fz.compress(Field(dims, smooth_trig_host(dims, s)), EB, preset) for s in range(3)]
    arcs.append(arcs[0])
    for a in arcs:
        for _ in range(2):
            assert fz.decompress_via_graph(a).data.tobytes() == fz.decompress(a).data.tobytes()
    # same sizes, different payload: scale the field by a power of two (codes
    # identical, outlier values and the header range differ) -> a graph hit
    f = Field(dims, smooth_trig_host(dims, 0))
    a0 = fz.compress(f, EB, preset)
    a1 = fz.compress(Field(dims, f.data * np.float32(2.0)), EB, preset)
    assert [len(p) for _, p in a0.segments] == [len(p) for _, p in a1.segments]
    for a in (a0, a1, a0):
        assert fz.decompress_via_graph(a).data.tobytes() == fz.decompress(a).data.tobytes()


def test_graph_cache_survives_buffer_growth():
    # graph A captured, a larger shape B grows the cached
    # buffers, then A replays -- it must still use live buffers
    a_dims, b_dims = (20, 30, 40), (40, 60, 80)
    fa, fb = (Field(d, smooth_trig_host(d, 5)) for d in (a_dims, b_dims))
    for preset in ("default", "speed"):
        ref_a = fz.serialize_archive(fz.compress(fa, EB, preset))
        ref_b = fz.serialize_archive(fz.compress(fb, EB, preset))
        for f, ref in ((fa, ref_a), (fb, ref_b), (fa, ref_a), (fb, ref_b)):
            a = fz.compress_via_graph(f, EB, preset)
            assert fz.serialize_archive(a) == ref
            assert fz.decompress_via_graph(a).data.tobytes() == fz.decompress(a).data.tobytes()


def test_device_archive_pickles_as_bytes():
    # payloads are views into a pinned block
    f = Field((16, 20, 24), smooth_trig_host((16, 20, 24), 4))
    a = fz.compress(f, EB, "default")
    for b in (pickle.loads(pickle.dumps(a)), copy.deepcopy(a)):
        assert fz.serialize_archive(b) == fz.serialize_archive(a)
        assert all(isinstance(p, bytes) for _, p in b.segments)
    assert isinstance(a.segment(2), bytes)


def test_decode_error_names_failing_stage():
    # a truncated Huffman stream fails in "decode-codes"; a broken outlier
    # segment in "decode-outliers" (pipeline.py:461-462 stage names)
    f = Field((16, 20, 24), smooth_trig_host((16, 20, 24), 6))
    a = fz.compress(f, EB, "default")
    segs = list(a.segments)
    k = [i for i, (kind, _) in enumerate(segs) if kind == 1][0]   # Huffman bitstream
    bad = fz.Archive(a.pipeline_id, a.eb_mode, a.eb_magnitude, a.data_min, a.data_max, a.dims, a.radius,
                     tuple(segs[:k] + [(1, bytes(segs[k][1])[:-3])] + segs[k + 1:]))
    with pytest.raises(E.StageError) as ei:
        fz.decompress(bad)
    assert ei.value.stage == "decode-codes"
    bad2 = fz.Archive(a.pipeline_id, a.eb_mode, a.eb_magnitude, a.data_min, a.data_max, a.dims, a.radius,
                      tuple([(2, b"\x01\x02\x03")] + segs[1:]))
    with pytest.raises(E.StageError) as ei:
        fz.decompress(bad2)
    assert ei.value.stage == "decode-outliers"
