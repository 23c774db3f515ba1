"""Host-side logic that needs no GPU: container format, pipeline specs,
secondary codec, generators -- checked against reference fixtures/oracle."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2509_20563_b200 import core, errors as E, secondary
from paper_2509_20563_b200.pipeline import PipelineSpec, StageKind, StageSpec, get_pipeline

ARCH = np.load(os.path.join(GOLDEN, "archives.npz"))


@pytest.mark.parametrize("name", list(ARCH["names"]))
@pytest.mark.parametrize("preset", ["default", "speed", "quality"])
def test_parse_serialize_round_trip_reference_archives(name, preset):
    blob = ARCH[f"{name}__{preset}__archive"].tobytes()
    a = core.parse_archive(blob)
    assert core.serialize_archive(a) == blob
    assert a.element_count == int(np.prod(ARCH[f"{name}__dims"]))


def test_header_is_41_bytes_and_constant_archive():
    a = core.Archive(0, core.ErrorMode.VALUE_RANGE_RELATIVE, 1e-3, 1.5, 1.5, (4, 5), 512, ())
    b = core.serialize_archive(a)
    assert len(b) == 41 and b[:4] == b"FZM1"
    assert core.parse_archive(b) == a


@pytest.mark.parametrize("mutate,exc", [
    (lambda b: b[:3], E.Truncated),
    (lambda b: b"XXXX" + b[4:], E.BadMagic),
    (lambda b: b[:4] + bytes([2]) + b[5:], E.UnsupportedVersion),
    (lambda b: b[:5] + bytes([77]) + b[6:], E.UnknownPipelineId),
    (lambda b: b + b"\x00", E.Truncated),
    (lambda b: b[:-1], E.Truncated),
])
def test_parse_rejects_corruption(mutate, exc):
    blob = ARCH["smooth2d__default__archive"].tobytes()
    with pytest.raises(exc):
        core.parse_archive(mutate(blob))


def test_pipeline_spec_validation_and_presets():
    assert [s.name for s in get_pipeline("default").stages] == ["predict", "histogram", "encode"]
    assert get_pipeline("speed").primary_codec == "bitshuffle"
    assert get_pipeline(2).predictor == "interp"
    spec = PipelineSpec(9, (StageSpec("p", StageKind.PREDICT, {"predictor": "lorenzo"}),
                            StageSpec("e", StageKind.PRIMARY_CODEC, {"codec": "huffman"})))
    assert [s.kind for s in spec.stages] == [StageKind.PREDICT, StageKind.ANALYSIS, StageKind.PRIMARY_CODEC]
    with pytest.raises(E.InvalidStageOrder):
        PipelineSpec(9, (StageSpec("e", StageKind.PRIMARY_CODEC), StageSpec("p", StageKind.PREDICT)))
    with pytest.raises(E.MissingStage):
        PipelineSpec(9, (StageSpec("p", StageKind.PREDICT),))
    with pytest.raises(E.UnknownPipelineId):
        get_pipeline("nope")


@pytest.mark.parametrize("data", [b"", b"\x00" * 10, b"abc", b"a\x00\x00\x00\x00b" * 50, bytes(range(256)) * 3,
                                  b"\x00\x00\x00x" * 100])
def test_zero_rle_round_trip(data):
    enc = secondary.zero_rle_encode(data)
    assert secondary.zero_rle_decode(enc) == data
    assert secondary.secondary_decode(secondary.secondary_encode(data)) == data


def test_zero_rle_matches_reference_format():
    # 5 zero bytes -> control 0 + LEB128(5); 3 literals -> 0x03 + bytes
    assert secondary.zero_rle_encode(b"\x00" * 5) == b"\x00\x05"
    assert secondary.zero_rle_encode(b"ab\x00") == b"\x03ab\x00"
    assert secondary.zero_rle_encode(b"\x00" * 300) == b"\x00\xac\x02"


def test_host_generators_match_oracle_definitions():
    from paper_2509_20563_b200 import data
    pred = np.load(os.path.join(GOLDEN, "predict.npz"))
    assert data.smooth_trig_host((17, 18, 19), 3).tobytes() == pred["smooth3d__orig"].tobytes()
    assert data.particle1d_host(50000, 0).tobytes() == pred["particle1d__orig"].tobytes()


def test_cpu_only_box_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2509_20563_b200 import compress, ErrorBoundSpec, ErrorMode, Field
    f = Field((8,), np.arange(8, dtype=np.float32))
    with pytest.raises(E.DeviceUnavailable):
        compress(f, ErrorBoundSpec(ErrorMode.ABSOLUTE, 0.1), "default")


@pytest.mark.parametrize("n", [1, 5, 8, 128, 129, 1000, 100_003])
def test_pairwise_tree_matches_numpy(n):
    # the split tree quality_device folds must reproduce numpy's summation
    from paper_2509_20563_b200.metrics import _pairwise_tree
    x = np.random.default_rng(n).random(n)
    off, ln, levels = _pairwise_tree(n)
    assert int(ln.astype(np.int64).sum()) == n and ln.max() <= 128

    def leaf(o, m):
        a = x[o:o + m]
        if m < 8:
            r = 0.0
            for v in a:
                r += v
            return r
        r = list(a[:8])
        full = m - m % 8
        for i in range(8, full, 8):
            for j in range(8):
                r[j] += a[i + j]
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        for i in range(full, m):
            res += a[i]
        return res

    ls = np.array([leaf(int(o), int(m)) for o, m in zip(off, ln)])
    below = None
    for lm, ids in reversed(levels):
        vals = np.empty(lm.size)
        vals[lm] = ls[ids]
        if below is not None:
            vals[~lm] = below[0::2] + below[1::2]
        below = vals
    assert below[0] == np.add.reduce(x)


@pytest.mark.parametrize("preset", ["default", "speed", "quality"])
def test_zero_copy_parse_and_wire_block(preset):
    # parse_archive of a read-only view keeps the payloads as views (no copy)
    # and round-trips; attach_wire lays an archive out exactly as
    # serialize_archive does, so archive_buffer needs no host assembly
    name = list(ARCH["names"])[0]
    blob = ARCH[f"{name}__{preset}__archive"].tobytes()
    view = memoryview(blob).toreadonly()
    a = core.parse_archive(view)
    assert all(isinstance(p, memoryview) for _, p in a.segments)
    assert core.serialize_archive(a) == blob
    assert a == core.parse_archive(blob)
    b = core.parse_archive(blob)
    head = len(core.header_bytes(b))
    block = np.zeros(len(blob), np.uint8)
    block[head:] = np.frombuffer(b"".join(bytes(p) for _, p in b.segments), np.uint8)
    core.attach_wire(b, block, head)
    assert bytes(core.archive_buffer(b)) == blob
    assert core.serialize_archive(b) == blob
    # a mutable buffer is copied once, as the reference does
    c = core.parse_archive(bytearray(blob))
    assert all(isinstance(p, bytes) for _, p in c.segments)
