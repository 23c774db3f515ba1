"""Pin the CPU oracle against fixtures produced by the reference fzpipe.

tests/golden/*.npz come from scripts/make_golden.py (reference run in the
build container).  Everything here must hold bit for bit.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN


def _load(name):
    return np.load(os.path.join(GOLDEN, name))


PRED = _load("predict.npz")
ARCH = _load("archives.npz")
BOOKS = _load("codebooks.npz")


@pytest.mark.parametrize("name", list(PRED["names"]))
def test_lorenzo_matches_reference(oracle, name):
    g = lambda k: PRED[f"{name}__{k}"]
    dims, eb, radius = tuple(g("dims")), float(g("eb")[0]), int(g("radius")[0])
    codes, idx, vals, recon = oracle.lorenzo_quantize(g("orig"), dims, eb, radius)
    assert np.array_equal(codes, g("lz_codes"))
    assert np.array_equal(idx, g("lz_oidx"))
    assert g("lz_oval").tobytes() == vals.tobytes()
    assert recon.tobytes() == g("lz_recon").tobytes()
    dec = oracle.lorenzo_reconstruct(codes, idx, vals, dims, eb, radius)
    assert dec.tobytes() == recon.tobytes()


@pytest.mark.parametrize("name", [n for n in PRED["names"] if f"{n}__ip_codes" in PRED])
def test_interp_matches_reference(oracle, name):
    g = lambda k: PRED[f"{name}__{k}"]
    dims, eb, radius = tuple(g("dims")), float(g("eb")[0]), int(g("radius")[0])
    codes, idx, vals, recon, anchors = oracle.interp_quantize(g("orig"), dims, eb, radius)
    assert np.array_equal(codes, g("ip_codes"))
    assert np.array_equal(idx, g("ip_oidx"))
    assert vals.tobytes() == g("ip_oval").tobytes()
    assert recon.tobytes() == g("ip_recon").tobytes()
    assert anchors == g("ip_anchors").tobytes()
    dec = oracle.interp_reconstruct(codes, idx, vals, anchors, dims, eb, radius)
    assert dec.tobytes() == recon.tobytes()


def test_package_merge_matches_reference(oracle):
    off = 0
    for nsym in BOOKS["sizes"]:
        h = BOOKS["hist"][off:off + nsym]
        want = BOOKS["lengths"][off:off + nsym]
        assert np.array_equal(oracle.code_lengths(h), want)
        off += nsym


@pytest.mark.parametrize("name", list(ARCH["names"]))
@pytest.mark.parametrize("preset", ["default", "speed", "quality"])
def test_archive_bytes_match_reference(oracle, name, preset):
    g = lambda k: ARCH[f"{name}__{k}"]
    dims = tuple(int(d) for d in g("dims"))
    blob = oracle.compress(g("orig"), dims, int(g("mode")[0]), float(g("mag")[0]), preset)
    assert blob == g(f"{preset}__archive").tobytes()
    rdims, rec = oracle.decompress(blob)
    assert tuple(rdims) == dims
    assert rec.tobytes() == g(f"{preset}__recon").tobytes()


def test_kats(oracle):
    # test_predict.py:28-47, test_encode.py:118-138, 220-227 of the reference suite.
    c, i, v, r = oracle.lorenzo_quantize(np.array([0, 1, 2], np.float32), (3,), 0.5)
    assert c.tolist() == [512, 513, 513] and i.size == 0 and r.tolist() == [0, 1, 2]
    codes = np.full(100, 7, np.uint32)
    cl, stream, bits = oracle.huffman_encode(codes, oracle.histogram(codes, 8))
    assert bits == 100 and len(stream) == 13 and cl[7] == 1
    assert np.array_equal(oracle.huffman_decode(cl, stream, 100), codes)
    codes = np.concatenate([np.full(c, s, np.uint32) for s, c in enumerate([4, 2, 1, 1])])
    cl, stream, bits = oracle.huffman_encode(codes, oracle.histogram(codes, 2))
    assert bits == 14
    bm, pay = oracle.bitshuffle_encode(np.ones(256, np.uint32), 512)
    assert np.frombuffer(pay, "<u4").tolist() == [0xFFFFFFFF] * 8
