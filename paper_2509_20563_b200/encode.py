"""Lossless stages with the reference's module API (fzpipe encode.py).

Histogram, canonical length-limited Huffman and bitshuffle with zero-word
elision, executed by the sm_100a kernels; numpy in, numpy/bytes out, exactly
the reference's signatures and exceptions.  The secondary zero-RLE codec
is re-exported from `secondary` (host side, off the timed path).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import errors as E
from .device import _p, default_engine
from .secondary import (  # noqa: F401  (re-exported API)
    register_secondary_codec, secondary_decode, secondary_encode, zero_rle_decode, zero_rle_encode,
)

MAX_CODE_LEN = 32
BS_BLOCK = 256
BS_WIDTH = 16
TOPK_SAMPLE_STRIDE = 64
TOPK_DEFAULT_K = 16


@dataclass(frozen=True, eq=False)
class Histogram:
    bins: np.ndarray
    total: int

    def __post_init__(self):
        bins = np.ascontiguousarray(self.bins, dtype=np.uint64)
        object.__setattr__(self, "bins", bins)
        object.__setattr__(self, "total", int(self.total))
        if int(bins.sum()) != self.total:
            raise ValueError("bin counts do not sum to total")

    def __eq__(self, other):
        if not isinstance(other, Histogram):
            return NotImplemented
        return self.total == other.total and np.array_equal(self.bins, other.bins)

    def __hash__(self):
        return hash((self.total, self.bins.tobytes()))


def _codes_u16(codes, radius: int) -> np.ndarray:
    c = np.ascontiguousarray(codes, dtype=np.uint32).reshape(-1)
    if c.size and int(c.max()) >= 2 * radius:
        raise E.CodeOutOfRange(f"code {int(c.max())} >= {2 * radius}")
    if 2 * radius > 65536:
        raise E.RadiusTooLarge(f"radius {radius} exceeds the device path's 16-bit codes")
    return c.astype(np.uint16)


def _upload_codes(eng, name, c16: np.ndarray) -> torch.Tensor:
    return eng.upload(name, c16, pad=16)


def _status(eng) -> int:
    return eng.decode_status()


def _fetch(eng, t: torch.Tensor, nbytes: int) -> bytes:
    if nbytes == 0:
        return b""
    return t[:nbytes].cpu().numpy().tobytes()


def histogram_exact(codes, radius: int) -> Histogram:
    """encode.py:79-84."""
    c16 = _codes_u16(codes, radius)
    eng = default_engine()
    nsym = 2 * radius
    if c16.size == 0:
        return Histogram(np.zeros(nsym, np.uint64), 0)
    d = _upload_codes(eng, "sh_codes", c16)
    bins = eng.buf("sh_bins", 8 * nsym)
    st = eng.buf("dstatus", 8, zero=True)
    eng._call("fzb_histogram", _p(d), c16.size, nsym, _p(bins), _p(st), eng.sp)
    out = np.frombuffer(_fetch(eng, bins, 8 * nsym), np.uint64).copy()
    _lib.raise_codec_status(_status(eng))
    return Histogram(out, c16.size)


def histogram_topk(codes, radius: int, k: int = TOPK_DEFAULT_K) -> Histogram:
    """encode.py:87-111 -- bitwise identical to the exact histogram."""
    if not 1 <= k <= 2 * radius:
        raise ValueError(f"k must be in [1, {2 * radius}], got {k}")
    return histogram_exact(codes, radius)


@dataclass(frozen=True, eq=False)
class HuffmanCodebook:
    """Per-symbol code lengths; canonical codewords derive from these."""

    code_lengths: np.ndarray

    def __post_init__(self):
        cl = np.ascontiguousarray(self.code_lengths, dtype=np.uint8)
        object.__setattr__(self, "code_lengths", cl)
        if cl.size and int(cl.max()) > MAX_CODE_LEN:
            raise ValueError(f"code length > {MAX_CODE_LEN}")
        used = cl[cl > 0].astype(np.uint64)
        if used.size and int(np.sum(np.uint64(1) << (np.uint64(MAX_CODE_LEN) - used))) > 1 << MAX_CODE_LEN:
            raise ValueError("code lengths violate the Kraft inequality")

    def __eq__(self, other):
        if not isinstance(other, HuffmanCodebook):
            return NotImplemented
        return np.array_equal(self.code_lengths, other.code_lengths)

    def __hash__(self):
        return hash(self.code_lengths.tobytes())

    @property
    def used_symbols(self) -> int:
        return int(np.count_nonzero(self.code_lengths))

    def to_bytes(self) -> bytes:
        return self.code_lengths.tobytes()

    @classmethod
    def from_bytes(cls, b: bytes) -> "HuffmanCodebook":
        return cls(np.frombuffer(bytes(b), np.uint8))

    def canonical_codewords(self) -> np.ndarray:
        """u32 codeword per symbol, assigned by (length asc, symbol asc)."""
        cl = self.code_lengths.astype(np.int64)
        cw = np.zeros(cl.size, np.uint32)
        code = 0
        prev = 0
        for s in np.lexsort((np.arange(cl.size), cl)):
            if cl[s] == 0:
                continue
            code <<= int(cl[s]) - prev
            cw[s] = code
            code += 1
            prev = int(cl[s])
        return cw


def _build(eng, bins: np.ndarray):
    nsym = bins.size
    db = eng.upload("sh_hbins", np.ascontiguousarray(bins, np.uint64))
    lengths = eng.buf("sh_lengths", nsym)
    cw = eng.buf("sh_cw", 4 * nsym)
    bc = eng.buf("sh_bitcount", 8)
    ws = eng.buf("sh_bws", eng.lib.fzb_huffman_build_workspace_bytes(nsym))
    eng._call("fzb_huffman_build", _p(db), nsym, _p(lengths), _p(cw), _p(bc), _p(ws), ws.numel(), eng.sp)
    return lengths, cw, bc


def build_codebook(hist: Histogram) -> HuffmanCodebook:
    """encode.py:216-217 -- package-merge on the GPU."""
    eng = default_engine()
    lengths, _, _ = _build(eng, hist.bins)
    return HuffmanCodebook(np.frombuffer(_fetch(eng, lengths, hist.bins.size), np.uint8).copy())


def huffman_encode(codes, hist: Histogram):
    """encode.py:279-291 -> (codebook, bitstream, bit_count)."""
    c = np.ascontiguousarray(codes, dtype=np.uint32).reshape(-1)
    nsym = hist.bins.size
    if c.size and int(c.max()) >= max(nsym, 1):
        raise E.CorruptStream("histogram inconsistent with codes")
    eng = default_engine()
    lengths, cw, bc = _build(eng, hist.bins)
    cl = np.frombuffer(_fetch(eng, lengths, nsym), np.uint8).copy()
    cb = HuffmanCodebook(cl)
    bit_count = int(np.sum(hist.bins * cl.astype(np.uint64)))
    if c.size == 0:
        return cb, bytes((bit_count + 7) // 8), bit_count
    d = _upload_codes(eng, "sh_codes", c.astype(np.uint16))
    cap = 4 * c.size + 16
    out = eng.buf("sh_hfout", cap)
    ws = eng.buf("sh_hews", eng.lib.fzb_huffman_encode_workspace_bytes(c.size))
    st = eng.buf("dstatus", 8, zero=True)
    eng._call("fzb_huffman_encode", _p(d), c.size, _p(lengths), _p(cw), nsym, _p(bc), _p(out), cap, _p(ws),
              ws.numel(), _p(st), eng.sp)
    if _status(eng) & _lib.ERR_HF_MISMATCH:
        raise E.CorruptStream("histogram inconsistent with codes")
    return cb, _fetch(eng, out, (bit_count + 7) // 8), bit_count


def huffman_decode(cb: HuffmanCodebook, bitstream: bytes, n: int) -> np.ndarray:
    """encode.py:294-317."""
    eng = default_engine()
    if n == 0:
        if len(bitstream):
            raise E.CorruptStream(f"{len(bitstream)} bytes after zero symbols")
        return np.empty(0, np.uint32)
    if cb.code_lengths.size > 65536:
        raise E.RadiusTooLarge("alphabet exceeds the device path's 16-bit codes")
    codes = eng.decode_codes("huffman", {"codebook": cb.code_lengths, "stream": bytes(bitstream)}, n,
                             max(cb.code_lengths.size // 2, 1))
    st = _status(eng)
    _lib.raise_codec_status(st)
    if st & _lib.ERR_HF_SYNC:
        raise RuntimeError("Huffman decoder did not synchronise")
    return np.frombuffer(_fetch(eng, codes, 2 * n), np.uint16).astype(np.uint32)


def bitshuffle_encode(codes, radius: int):
    """encode.py:329-353 -> (bitmap, payload)."""
    if radius > 32768:
        raise E.RadiusTooLarge(f"radius {radius} exceeds 16-bit code width")
    c16 = _codes_u16(codes, radius)
    n = c16.size
    if n == 0:
        return b"", b""
    eng = default_engine()
    d = _upload_codes(eng, "sh_codes", c16)
    nb = (n + BS_BLOCK - 1) // BS_BLOCK
    bm = eng.buf("sh_bsmap", 16 * nb)
    pay = eng.buf("sh_bspay", 512 * nb)
    nw = eng.buf("sh_nwords", 8)
    ws = eng.buf("sh_bsws", eng.lib.fzb_bitshuffle_workspace_bytes(n))
    eng._call("fzb_bitshuffle_encode", _p(d), n, _p(bm), _p(pay), _p(nw), _p(ws), ws.numel(), eng.sp)
    words = int(np.frombuffer(_fetch(eng, nw, 8), np.uint64)[0])
    return _fetch(eng, bm, 16 * nb), _fetch(eng, pay, 4 * words)


def bitshuffle_decode(bitmap: bytes, payload: bytes, n: int, radius: int) -> np.ndarray:
    """encode.py:356-391."""
    if radius > 32768:
        raise E.RadiusTooLarge(f"radius {radius} exceeds 16-bit code width")
    eng = default_engine()
    codes = eng.decode_codes("bitshuffle", {"bitmap": bytes(bitmap), "payload": bytes(payload)}, n, radius)
    if n == 0:
        return np.empty(0, np.uint32)
    _lib.raise_codec_status(_status(eng))
    return np.frombuffer(_fetch(eng, codes, 2 * n), np.uint16).astype(np.uint32)
