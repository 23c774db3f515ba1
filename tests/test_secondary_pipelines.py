"""Pipelines with a secondary-codec stage (reference
pipeline.py:307-312 wrap, 390-399 unwrap; encode.py:426-516 zero-RLE).

Fixtures: tests/golden/secondary.npz, made by the REFERENCE fzpipe through
custom pipelines 60 (lorenzo + bitshuffle + secondary 0), 61 (lorenzo +
huffman + secondary 0) and 62 (interp + huffman + secondary 0)
(scripts/make_secondary_golden.py).

CPU: the host secondary codec unwraps every fixture segment to exactly the
primary segments the oracle produces for the matching preset, and re-wraps
them to the fixture's bytes.  GPU: the same custom pipelines registered in
this package compress the fixture inputs to byte-identical archives and
decompress fzpipe's archives to its reconstructions."""

import os

import numpy as np
import pytest

from conftest import GOLDEN

G = np.load(os.path.join(GOLDEN, "secondary.npz"))
NAMES = list(G["names"])
PRESET_OF = {("lorenzo", "bitshuffle"): "speed", ("lorenzo", "huffman"): "default", ("interp", "huffman"): "quality"}


def _spec_of(pid):
    i = list(G["spec_ids"]).index(pid)
    return str(G["spec_pred"][i]), str(G["spec_codec"][i])


@pytest.fixture(autouse=True, scope="module")
def _registered():
    """The custom pipelines, registered in this package (host-side registry)."""
    from paper_2509_20563_b200.pipeline import PipelineSpec, StageKind, StageSpec, register_pipeline
    for pid in G["spec_ids"]:
        pred, codec = _spec_of(int(pid))
        register_pipeline(PipelineSpec(int(pid), (
            StageSpec("predict", StageKind.PREDICT, {"predictor": pred}),
            StageSpec("encode", StageKind.PRIMARY_CODEC, {"codec": codec}),
            StageSpec("shrink", StageKind.SECONDARY_CODEC, {"codec_id": "0"}),
        )))


@pytest.mark.parametrize("name", NAMES)
def test_secondary_wrap_matches_oracle_segments(oracle, name):
    from paper_2509_20563_b200 import secondary
    from paper_2509_20563_b200.core import SEG_SECONDARY_WRAPPED, parse_archive
    pid = int(G[f"{name}__pid"][0])
    dims = tuple(int(d) for d in G[f"{name}__dims"])
    a = parse_archive(G[f"{name}__archive"].tobytes())
    assert a.pipeline_id == pid
    want = oracle.parse(oracle.compress(G[f"{name}__orig"], dims, 1, float(G[f"{name}__rel"][0]),
                                       PRESET_OF[_spec_of(pid)]))["segments"]
    got = []
    for kind, payload in a.segments:
        if kind == SEG_SECONDARY_WRAPPED:
            inner = secondary.secondary_decode(payload[1:])
            got.append((payload[0], inner))
            assert payload == bytes([payload[0]]) + secondary.secondary_encode(inner, 0)   # the wrap is byte-exact
        else:
            got.append((kind, bytes(payload)))
    assert [(k, bytes(p)) for k, p in want] == got


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_secondary_pipeline_byte_identical(name):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2509_20563_b200 as fz
    pid = int(G[f"{name}__pid"][0])
    dims = tuple(int(d) for d in G[f"{name}__dims"])
    f = fz.Field(dims, G[f"{name}__orig"])
    a = fz.compress(f, fz.ErrorBoundSpec(fz.ErrorMode.VALUE_RANGE_RELATIVE, float(G[f"{name}__rel"][0])), pid)
    assert fz.serialize_archive(a) == G[f"{name}__archive"].tobytes()
    r = fz.decompress(fz.parse_archive(G[f"{name}__archive"].tobytes()))
    assert r.data.tobytes() == G[f"{name}__recon"].tobytes()
