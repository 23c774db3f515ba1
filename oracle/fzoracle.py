"""CPU oracle for the FZModules hot path -- TEST INFRASTRUCTURE ONLY.

A restatement of the reference `fzpipe` (arXiv 2509.20563's CPU reference,
/root/reference/pkg/src/fzpipe) used to check the B200 kernels.  The
arithmetic lives in fzoracle.c (ctypes); this module restates the host-side
glue: the predictor wrappers (predict.py:221-344), the codec wrappers
(encode.py:79-391) and the sequential compress/decompress executor with its
container format (pipeline.py:300-470, core.py:285-374).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this module.  The product package never does.
Pinned against fzpipe itself via tests/golden/ (scripts/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import struct
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_BUILD = os.path.join(_HERE, "_build")
_SO = os.path.join(_BUILD, "libfzoracle.so")

MAGIC = b"FZM1"
_HDR = struct.Struct("<4s4Bd2f3IIB")  # core.py:56 (41 bytes)
_SEG = struct.Struct("<BQ")  # core.py:57
SEG_HF_BOOK, SEG_HF_STREAM, SEG_OUT_IDX, SEG_OUT_VAL, SEG_BS_MAP, SEG_BS_PAY, SEG_ANCHOR = range(7)
SEG_DQ_DELTAS = 8   # opt-in dual-quant pipelines only (this repo's own format, not the reference's)
SEG_INTERP_PROFILE = 9   # opt-in profiled G-Interp (pipeline 5): [anchor stride, weights id]

# preset table, pipeline.py:200-214: id -> (predictor, codec); ids 3/4 are the
# opt-in dual-quant pipelines of this repo (no reference counterpart; checked
# against dq_quantize / dq_reconstruct below, a numpy statement of their spec)
PRESETS = {0: ("lorenzo", "huffman"), 1: ("lorenzo", "bitshuffle"), 2: ("interp", "huffman"),
           3: ("dualquant", "bitshuffle"), 4: ("dualquant", "huffman"), 5: ("interp-profiled", "huffman")}
PRESET_NAMES = {"default": 0, "speed": 1, "quality": 2, "dq-speed": 3, "dq-default": 4, "q-profiled": 5}
# profiled G-Interp candidates (csrc/interp.cu interp_profile_kernel): c = 3 s + w
PROFILE_STRIDES = (16, 8)
PROFILE_WEIGHTS = ((-0.0625, 0.5625, 0.5625, -0.0625), (0.0, 0.5, 0.5, 0.0), (-0.075, 0.575, 0.575, -0.075))
CUBIC = (-1 / 16, 9 / 16, 9 / 16, -1 / 16)  # predict.py:47


class OracleError(Exception):
    """Carries the fzpipe error class name the reference would raise."""

    def __init__(self, kind: str, msg: str = ""):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


def build(force: bool = False) -> str:
    """Compile fzoracle.c with gcc (no FMA contraction, IEEE math)."""

    src = os.path.join(_HERE, "fzoracle.c")
    if not force and os.path.exists(_SO) and os.path.getmtime(_SO) >= os.path.getmtime(src):
        return _SO
    os.makedirs(_BUILD, exist_ok=True)
    cmd = ["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
           "-fvisibility=hidden", "-o", _SO + ".tmp", src, "-lm"]
    subprocess.check_call(cmd)
    os.replace(_SO + ".tmp", _SO)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        D = ctypes.c_double
        L.fzo_minmax.argtypes = [P, I64, P, P]
        L.fzo_lorenzo_encode.argtypes = [P, P, P, P, I64, I64, I64, D, I64]
        L.fzo_lorenzo_decode.argtypes = [P, P, P, I64, I64, I64, D, I64]
        L.fzo_interp_run.argtypes = [P, P, P, P, I64, I64, I64, D, I64, I64, P, ctypes.c_int]
        L.fzo_histogram.argtypes = [P, I64, I64, P]
        L.fzo_histogram.restype = ctypes.c_int
        L.fzo_package_merge.argtypes = [P, I64, ctypes.c_int, P]
        L.fzo_package_merge.restype = ctypes.c_int
        L.fzo_canonical_codewords.argtypes = [P, I64, P]
        L.fzo_huffman_pack.argtypes = [P, I64, P, P, P]
        L.fzo_huffman_pack.restype = I64
        L.fzo_huffman_unpack.argtypes = [P, I64, I64, P, I64, P]
        L.fzo_huffman_unpack.restype = I64
        L.fzo_bitshuffle_encode.argtypes = [P, I64, P, P]
        L.fzo_bitshuffle_encode.restype = I64
        L.fzo_bitshuffle_decode.argtypes = [P, P, I64, I64, P]
        L.fzo_bitshuffle_decode.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def pad3(dims):
    """predict.py:204-205."""
    dims = tuple(int(d) for d in dims)
    return (1,) * (3 - len(dims)) + dims


# ------------------------------------------------------------------ bound

def minmax(data: np.ndarray) -> tuple[float, float]:
    lo = np.zeros(1, np.float32)
    hi = np.zeros(1, np.float32)
    lib().fzo_minmax(_p(data), data.size, _p(lo), _p(hi))
    return float(lo[0]), float(hi[0])


def resolve_eb(eb_mode: int, magnitude: float, lo: float, hi: float) -> float:
    """core.py:155-170 (relative: magnitude * (hi - lo) in f64)."""
    if eb_mode == 1:
        if hi == lo:
            raise OracleError("ZeroRange")
        return float(magnitude) * (hi - lo)
    return float(magnitude)


# -------------------------------------------------------------- predictors

def lorenzo_quantize(data: np.ndarray, dims, eb: float, radius: int = 512):
    """predict.py:221-239 -> (codes u32, outlier idx i64, outlier vals f32, recon f32)."""
    data = np.ascontiguousarray(data, np.float32).reshape(-1)
    n0, n1, n2 = pad3(dims)
    codes = np.empty(data.size, np.uint32)
    recon = np.zeros(data.size, np.float32)
    flags = np.zeros(data.size, np.uint8)
    lib().fzo_lorenzo_encode(_p(data), _p(codes), _p(recon), _p(flags), n0, n1, n2, float(eb), int(radius))
    idx = np.nonzero(flags)[0].astype(np.int64)
    return codes, idx, data[idx].astype(np.float32), recon


def _check_decode_codes(codes, radius):
    if codes.size and int(codes.max()) >= 2 * radius:
        raise OracleError("MalformedCodes", "code >= 2*radius")


def lorenzo_reconstruct(codes, idx, vals, dims, eb: float, radius: int = 512) -> np.ndarray:
    """predict.py:242-253."""
    codes = np.ascontiguousarray(codes, np.uint32)
    _check_decode_codes(codes, radius)
    n0, n1, n2 = pad3(dims)
    recon = np.zeros(codes.size, np.float32)
    flags = np.zeros(codes.size, np.uint8)
    recon[idx] = vals
    flags[idx] = 1
    lib().fzo_lorenzo_decode(_p(codes), _p(flags), _p(recon), n0, n1, n2, float(eb), int(radius))
    return recon


def interp_applicable(dims, anchor_stride: int = 16) -> bool:
    """predict.py:264-267."""
    if len(dims) == 1:
        return False
    return all(d >= anchor_stride + 1 for d in dims)


def interp_quantize(data, dims, eb: float, radius: int = 512, anchor_stride: int = 16, weights=CUBIC):
    """predict.py:270-306 -> (codes, idx, vals, recon, anchor bytes)."""
    data = np.ascontiguousarray(data, np.float32).reshape(-1)
    if not interp_applicable(dims, anchor_stride):
        c, i, v, r = lorenzo_quantize(data, dims, eb, radius)
        return c, i, v, r, b""
    n0, n1, n2 = pad3(dims)
    a = anchor_stride
    codes = np.full(data.size, int(radius), np.uint32)
    recon = np.zeros(data.size, np.float32)
    flags = np.zeros(data.size, np.uint8)
    anchors = np.ascontiguousarray(data.reshape(n0, n1, n2)[::a, ::a, ::a])
    recon.reshape(n0, n1, n2)[::a, ::a, ::a] = anchors
    w = np.array(weights, np.float64)
    lib().fzo_interp_run(_p(data), _p(codes), _p(recon), _p(flags), n0, n1, n2, float(eb),
                         int(radius), a, _p(w), 1)
    idx = np.nonzero(flags)[0].astype(np.int64)
    return codes, idx, data[idx].astype(np.float32), recon, anchors.astype("<f4").tobytes()


def interp_reconstruct(codes, idx, vals, anchors: bytes, dims, eb: float, radius: int = 512,
                       anchor_stride: int = 16, weights=CUBIC) -> np.ndarray:
    """predict.py:322-344."""
    if len(anchors) == 0:
        return lorenzo_reconstruct(codes, idx, vals, dims, eb, radius)
    codes = np.ascontiguousarray(codes, np.uint32)
    _check_decode_codes(codes, radius)
    n0, n1, n2 = pad3(dims)
    a = anchor_stride
    adims = tuple((d - 1) // a + 1 for d in (n0, n1, n2))
    if len(anchors) != 4 * adims[0] * adims[1] * adims[2]:
        raise OracleError("AnchorSizeMismatch")
    recon = np.zeros(codes.size, np.float32)
    flags = np.zeros(codes.size, np.uint8)
    recon[idx] = vals
    flags[idx] = 1
    recon.reshape(n0, n1, n2)[::a, ::a, ::a] = np.frombuffer(anchors, "<f4").reshape(adims)
    w = np.array(weights, np.float64)
    empty = np.zeros(1, np.float32)
    lib().fzo_interp_run(_p(empty), _p(codes), _p(recon), _p(flags), n0, n1, n2, float(eb),
                         int(radius), a, _p(w), 0)
    return recon


# ------------------------------------------------------------------ codecs

# ------------------------------------------------- dual-quant (opt-in ids 3/4)
# Spec (paper_2509_20563_b200/csrc/dualquant.cu): p = rint(x * RN(1/2eb)) in f64
# (|.| < 2^27), delta = Lorenzo difference of p with zero padding, code =
# delta + R when |delta| < R and |RN32(2eb p) - x| <= eb, else an outlier
# (code R; the archive keeps index, original value and delta).

DQ_PMAX = 2.0 ** 27


def dq_quantize(data: np.ndarray, dims, eb: float, radius: int = 512):
    """-> (codes u32, outlier idx i64, values f32, deltas i32)."""
    x = np.ascontiguousarray(data, np.float32).reshape(pad3(dims))
    inv2eb = 1.0 / (2.0 * eb)
    q = x.astype(np.float64) * inv2eb
    if not (np.abs(q) < DQ_PMAX).all():
        raise OracleError("DualQuantRange")
    p = np.rint(q).astype(np.int64)
    pp = np.pad(p, ((1, 0), (1, 0), (1, 0)))
    d = (pp[1:, 1:, 1:] - pp[1:, :-1, 1:] - pp[1:, 1:, :-1] + pp[1:, :-1, :-1]
         - pp[:-1, 1:, 1:] + pp[:-1, :-1, 1:] + pp[:-1, 1:, :-1] - pp[:-1, :-1, :-1])
    rec = (2.0 * eb * p.astype(np.float64)).astype(np.float32)
    ok = (np.abs(d) < radius) & (np.abs(rec.astype(np.float64) - x.astype(np.float64)) <= eb)
    codes = np.where(ok, d + radius, radius).astype(np.uint32).reshape(-1)
    idx = np.flatnonzero(~ok.reshape(-1)).astype(np.int64)
    return codes, idx, x.reshape(-1)[idx].copy(), d.reshape(-1)[idx].astype(np.int32)


def dq_reconstruct(codes, idx, vals, deltas, dims, eb: float, radius: int = 512) -> np.ndarray:
    d = codes.astype(np.int64) - radius
    d[idx] = deltas
    p = d.reshape(pad3(dims)).cumsum(axis=2).cumsum(axis=1).cumsum(axis=0)
    rec = (2.0 * eb * p.astype(np.float64)).astype(np.float32).reshape(-1)
    rec[idx] = vals
    return rec


def interp_profile(data: np.ndarray, dims, eb: float) -> np.ndarray:
    """Sampled cost of the 6 (anchor stride, weights) candidates of pipeline 5
    (spec: csrc/interp.cu interp_profile_kernel) -> u64[6]."""
    n0, n1, n2 = pad3(dims)
    x = np.ascontiguousarray(data, np.float32).reshape(n0, n1, n2)
    inv2eb = 1.0 / (2.0 * eb)
    axes = [np.arange(n) for n in (n0, n1, n2)]
    sel = [a[((a >> 4) & 3) == 0] for a in axes]           # 16-cells whose cell coordinate is a multiple of 4
    I, J, K = np.meshgrid(*sel, indexing="ij")
    co = [I.reshape(-1), J.reshape(-1), K.reshape(-1)]
    xv = x[co[0], co[1], co[2]].astype(np.float64)

    def lowbit(c):
        c = c.astype(np.int64)
        out = np.full(c.shape, 62, np.int64)
        nz = c != 0
        out[nz] = np.log2(c[nz] & -c[nz]).astype(np.int64)
        return out

    lb = [lowbit(c) for c in co]
    m = np.minimum(lb[0], np.minimum(lb[1], lb[2]))
    ext = (n0, n1, n2)
    flat = x.reshape(-1)
    strides = (n1 * n2, n2, 1)
    t = (co[0] * n1 + co[1]) * n2 + co[2]
    scores = np.zeros(6, np.uint64)
    for s, A in enumerate(PROFILE_STRIDES):
        anchor = m >= int(np.log2(A))
        for wi in range(3):
            scores[3 * s + wi] += np.uint64(32 * int(anchor.sum()))
        tgt = ~anchor
        h = (1 << m[tgt]).astype(np.int64)
        ax = np.where(lb[2][tgt] == m[tgt], 2, np.where(lb[1][tgt] == m[tgt], 1, 0))
        c = np.choose(ax, [co[0][tgt], co[1][tgt], co[2][tgt]])
        n = np.choose(ax, list(ext))
        sh = h * np.choose(ax, list(strides))
        tt = t[tgt]
        cub = (c - 3 * h >= 0) & (c + 3 * h < n)
        lin = ~cub & (c + h < n)
        get = lambda off, ok: np.where(ok, flat[np.where(ok, tt + off, 0)], 0).astype(np.float64)
        for wi, W in enumerate(PROFILE_WEIGHTS):
            pc = W[0] * get(-3 * sh, cub)
            pc = pc + W[1] * get(-sh, cub)
            pc = pc + W[2] * get(sh, cub)
            pc = pc + W[3] * get(3 * sh, cub)
            pl = 0.5 * get(-sh, lin) + 0.5 * get(sh, lin)
            pcp = flat[tt - sh].astype(np.float64)
            pred = np.where(cub, pc, np.where(lin, pl, pcp))
            e = np.minimum(np.abs(pred - xv[tgt]) * inv2eb, 1073741824.0)
            iv = np.rint(e).astype(np.uint64)
            bits = np.zeros(iv.shape, np.uint64)
            nz = iv > 0
            bits[nz] = np.floor(np.log2(iv[nz].astype(np.float64))).astype(np.uint64) + 1
            scores[3 * s + wi] += np.uint64(int(bits.sum()))
    return scores


def profile_choice(scores) -> tuple:
    c = int(np.argmin(np.asarray(scores, np.uint64)))   # ties: the lowest index
    return PROFILE_STRIDES[c // 3], c % 3


def histogram(codes, radius: int) -> np.ndarray:
    """encode.py:79-84 (and topk 87-111, bitwise identical)."""
    codes = np.ascontiguousarray(codes, np.uint32)
    bins = np.zeros(2 * radius, np.uint64)
    if lib().fzo_histogram(_p(codes), codes.size, 2 * radius, _p(bins)) != 0:
        raise OracleError("CodeOutOfRange")
    return bins


def code_lengths(bins: np.ndarray, limit: int = 32) -> np.ndarray:
    """encode.py:174-217 (build_codebook)."""
    bins = np.ascontiguousarray(bins, np.uint64)
    out = np.zeros(bins.size, np.uint8)
    if lib().fzo_package_merge(_p(bins), bins.size, limit, _p(out)) != 0:
        raise MemoryError
    return out


def codewords(lengths: np.ndarray) -> np.ndarray:
    lengths = np.ascontiguousarray(lengths, np.uint8)
    cw = np.zeros(lengths.size, np.uint32)
    lib().fzo_canonical_codewords(_p(lengths), lengths.size, _p(cw))
    return cw


def huffman_encode(codes, bins):
    """encode.py:279-291 -> (lengths, stream bytes, bit count)."""
    codes = np.ascontiguousarray(codes, np.uint32)
    cl = code_lengths(bins)
    bit_count = int(np.sum(bins * cl.astype(np.uint64)))
    out = np.zeros((bit_count + 7) // 8, np.uint8)
    if codes.size:
        got = lib().fzo_huffman_pack(_p(codes), codes.size, _p(codewords(cl)), _p(cl), _p(out))
        if got != bit_count:
            raise OracleError("CorruptStream", "histogram inconsistent with codes")
    return cl, out.tobytes(), bit_count


def huffman_decode(lengths, stream: bytes, n: int) -> np.ndarray:
    """encode.py:294-317."""
    cl = np.ascontiguousarray(np.frombuffer(bytes(lengths), np.uint8) if isinstance(lengths, (bytes, bytearray)) else lengths, np.uint8)
    if cl.size and int(cl.max()) > 32:
        raise OracleError("ValueError", "code length > 32")
    used = cl[cl > 0].astype(np.uint64)
    if used.size and int(np.sum(np.uint64(1) << (np.uint64(32) - used))) > (1 << 32):
        raise OracleError("ValueError", "Kraft")
    s = np.frombuffer(stream, np.uint8)
    out = np.empty(n, np.uint32)
    if n == 0:
        if s.size:
            raise OracleError("CorruptStream", "bytes after zero symbols")
        return out
    if not cl.size or int(cl.max()) == 0:
        raise OracleError("CorruptStream", "empty codebook")
    s = np.ascontiguousarray(s)
    end = lib().fzo_huffman_unpack(_p(s), s.size, n, _p(cl), cl.size, _p(out))
    if end == -1:
        raise OracleError("Truncated")
    if end == -2:
        raise OracleError("CorruptStream", "no codeword")
    if s.size != (end + 7) // 8:
        raise OracleError("CorruptStream", "stream longer than needed")
    if end & 7 and int(s[-1]) & ((1 << (8 - (end & 7))) - 1):
        raise OracleError("CorruptStream", "nonzero padding")
    return out


def bitshuffle_encode(codes, radius: int):
    """encode.py:329-353 -> (bitmap, payload)."""
    if radius > 32768:
        raise OracleError("RadiusTooLarge")
    codes = np.ascontiguousarray(codes, np.uint32)
    if codes.size and int(codes.max()) >= 2 * radius:
        raise OracleError("CodeOutOfRange")
    nb = (codes.size + 255) // 256
    bitmap = np.zeros(nb * 16, np.uint8)
    payload = np.zeros(nb * 128, np.uint32)
    np_ = lib().fzo_bitshuffle_encode(_p(codes), codes.size, _p(bitmap), _p(payload))
    return bitmap.tobytes(), payload[:np_].astype("<u4").tobytes()


def bitshuffle_decode(bitmap: bytes, payload: bytes, n: int, radius: int) -> np.ndarray:
    """encode.py:356-391."""
    if radius > 32768:
        raise OracleError("RadiusTooLarge")
    nb = (n + 255) // 256
    nwords = nb * 128
    need = (nwords + 7) // 8
    if len(bitmap) < need:
        raise OracleError("Truncated")
    if len(bitmap) > need:
        raise OracleError("BitmapPayloadMismatch")
    bm = np.frombuffer(bitmap, np.uint8)
    if len(payload) % 4:
        raise OracleError("BitmapPayloadMismatch")
    marked = int(np.unpackbits(bm).sum()) if bm.size else 0
    if len(payload) // 4 != marked:
        raise OracleError("BitmapPayloadMismatch")
    pay = np.ascontiguousarray(np.frombuffer(payload, "<u4").astype(np.uint32))
    out = np.zeros(n, np.uint32)
    bm = np.ascontiguousarray(bm)
    if pay.size == 0:
        pay = np.zeros(1, np.uint32)
    rc = lib().fzo_bitshuffle_decode(_p(bm), _p(pay), n, int(radius), _p(out))
    if rc != 0:
        raise OracleError("CorruptPayload")
    return out


# --------------------------------------------------------------- container

def serialize(pipeline_id, eb_mode, magnitude, lo, hi, dims, radius, segments) -> bytes:
    """core.py:285-309."""
    d3 = list(dims) + [1] * (3 - len(dims))
    out = bytearray(_HDR.pack(MAGIC, 1, pipeline_id, eb_mode, len(dims), float(magnitude),
                              lo, hi, d3[0], d3[1], d3[2], radius, len(segments)))
    for k, p in segments:
        out += _SEG.pack(k, len(p))
    for _, p in segments:
        out += p
    return bytes(out)


def parse(b: bytes):
    """core.py:312-374 (structural checks)."""
    if len(b) < 4:
        raise OracleError("Truncated")
    if b[:4] != MAGIC:
        raise OracleError("BadMagic")
    if len(b) < _HDR.size:
        raise OracleError("Truncated")
    (_, ver, pid, mode, ndim, mag, lo, hi, d0, d1, d2, radius, nseg) = _HDR.unpack_from(b, 0)
    if ver != 1:
        raise OracleError("UnsupportedVersion")
    if pid not in PRESETS:
        raise OracleError("UnknownPipelineId")
    if not 1 <= ndim <= 3 or mode not in (0, 1):
        raise OracleError("ArchiveError")
    pos = _HDR.size + nseg * _SEG.size
    if len(b) < pos:
        raise OracleError("Truncated")
    ents = [_SEG.unpack_from(b, _HDR.size + i * _SEG.size) for i in range(nseg)]
    segs = []
    for k, ln in ents:
        if len(b) < pos + ln:
            raise OracleError("Truncated")
        segs.append((k, b[pos:pos + ln]))
        pos += ln
    if pos != len(b):
        raise OracleError("Truncated")
    return dict(pipeline_id=pid, eb_mode=mode, magnitude=mag, lo=lo, hi=hi,
                dims=(d0, d1, d2)[:ndim], radius=radius, segments=segs)


# ---------------------------------------------------------------- executor

def compress(data: np.ndarray, dims, eb_mode: int, magnitude: float, pipeline,
             radius: int = 512, anchor_stride: int = 16) -> bytes:
    """pipeline.py:345-379 for presets 0/1/2; returns serialized archive bytes."""
    pid = PRESET_NAMES[pipeline] if isinstance(pipeline, str) else int(pipeline)
    predictor, codec = PRESETS[pid]
    data = np.ascontiguousarray(data, np.float32).reshape(-1)
    dims = tuple(int(d) for d in dims)
    lo, hi = minmax(data)
    if lo == hi:
        return serialize(pid, eb_mode, magnitude, lo, hi, dims, radius, [])
    eb = resolve_eb(eb_mode, magnitude, lo, hi)
    deltas = None
    prof = None
    if predictor == "interp-profiled" and not interp_applicable(dims, 16):
        predictor = "interp"   # (the reference's 1D / small-extent fallback to Lorenzo, no profile)
    if predictor == "interp":
        codes, idx, vals, _, anchors = interp_quantize(data, dims, eb, radius, anchor_stride)
    elif predictor == "interp-profiled":
        stride, wi = profile_choice(interp_profile(data, dims, eb))
        prof = bytes([stride, wi])
        codes, idx, vals, _, anchors = interp_quantize(data, dims, eb, radius, stride, PROFILE_WEIGHTS[wi])
    elif predictor == "dualquant":
        codes, idx, vals, deltas = dq_quantize(data, dims, eb, radius)
        anchors = b""
    else:
        codes, idx, vals, _ = lorenzo_quantize(data, dims, eb, radius)
        anchors = b""
    segs = [(SEG_OUT_IDX, idx.astype("<u8").tobytes()), (SEG_OUT_VAL, vals.astype("<f4").tobytes())]
    if deltas is not None:
        segs.append((SEG_DQ_DELTAS, deltas.astype("<i4").tobytes()))
    if prof is not None:
        segs.append((SEG_INTERP_PROFILE, prof))
    if anchors:
        segs.append((SEG_ANCHOR, anchors))
    if codec == "huffman":
        cl, stream, _ = huffman_encode(codes, histogram(codes, radius))
        segs += [(SEG_HF_BOOK, cl.tobytes()), (SEG_HF_STREAM, stream)]
    else:
        bm, pay = bitshuffle_encode(codes, radius)
        segs += [(SEG_BS_MAP, bm), (SEG_BS_PAY, pay)]
    return serialize(pid, eb_mode, magnitude, lo, hi, dims, radius, segs)


def decompress(archive: bytes, anchor_stride: int = 16):
    """pipeline.py:439-466 -> (dims, f32 data)."""
    a = parse(archive)
    dims = a["dims"]
    n = int(np.prod(dims))
    predictor, codec = PRESETS[a["pipeline_id"]]
    if not a["segments"]:
        if a["lo"] != a["hi"]:
            raise OracleError("CorruptPayload")
        return dims, np.full(n, a["lo"], np.float32)
    lo32, hi32 = float(np.float32(a["lo"])), float(np.float32(a["hi"]))
    eb = a["magnitude"] * (hi32 - lo32) if a["eb_mode"] == 1 else a["magnitude"]
    segs = dict(a["segments"])
    radius = a["radius"]
    if codec == "huffman":
        if SEG_HF_BOOK not in segs or SEG_HF_STREAM not in segs:
            raise OracleError("CorruptPayload")
        cl = np.frombuffer(segs[SEG_HF_BOOK], np.uint8)
        if cl.size != 2 * radius:
            raise OracleError("CorruptPayload")
        codes = huffman_decode(cl, segs[SEG_HF_STREAM], n)
    else:
        if SEG_BS_MAP not in segs or SEG_BS_PAY not in segs:
            raise OracleError("CorruptPayload")
        codes = bitshuffle_decode(segs[SEG_BS_MAP], segs[SEG_BS_PAY], n, radius)
    if SEG_OUT_IDX not in segs or SEG_OUT_VAL not in segs:
        raise OracleError("CorruptPayload")
    ib, vb = segs[SEG_OUT_IDX], segs[SEG_OUT_VAL]
    if len(ib) % 8 or len(vb) % 4 or len(ib) // 8 != len(vb) // 4:
        raise OracleError("CorruptPayload")
    idx = np.frombuffer(ib, "<u8").astype(np.int64)
    vals = np.frombuffer(vb, "<f4").astype(np.float32)
    if idx.size and (int(idx.max()) >= n or int(idx.min()) < 0):
        raise OracleError("CorruptPayload")
    _check_decode_codes(codes, radius)
    if idx.size > 1 and not (np.diff(idx) > 0).all():
        raise OracleError("MalformedCodes")
    if idx.size and not (codes[idx] == radius).all():
        raise OracleError("MalformedCodes")
    anchors = segs.get(SEG_ANCHOR, b"")
    if predictor == "dualquant":
        db = segs.get(SEG_DQ_DELTAS)
        if db is None or len(db) != 4 * idx.size:
            raise OracleError("CorruptPayload")
        rec = dq_reconstruct(codes, idx, vals, np.frombuffer(db, "<i4"), dims, eb, radius)
    elif predictor in ("interp", "interp-profiled"):
        pb = segs.get(SEG_INTERP_PROFILE)
        if predictor == "interp-profiled" and pb is not None:
            if len(pb) != 2 or pb[0] not in PROFILE_STRIDES or pb[1] > 2:
                raise OracleError("CorruptPayload")
            rec = interp_reconstruct(codes, idx, vals, anchors, dims, eb, radius, pb[0], PROFILE_WEIGHTS[pb[1]])
        else:
            rec = interp_reconstruct(codes, idx, vals, anchors, dims, eb, radius, anchor_stride)
    else:
        rec = lorenzo_reconstruct(codes, idx, vals, dims, eb, radius)
    return dims, rec
