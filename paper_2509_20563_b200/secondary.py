"""Secondary byte codec stage (reference encode.py:394-516) -- host side.

Outside the timed path by the north star; kept so custom pipelines with a
SecondaryCodec stage round-trip byte-identically.  Codec 0 is the zero-run
coder: control 0x00 + LEB128 length for runs of >= 4 zero bytes, control
0x01..0xFE for that many literal bytes, 0xFF reserved.
"""

from __future__ import annotations

import numpy as np

from . import errors as E

_MIN_RUN = 4
_MAX_LIT = 254


def _leb(v: int) -> bytes:
    out = bytearray()
    while True:
        b, v = v & 0x7F, v >> 7
        out.append(b | (0x80 if v else 0))
        if not v:
            return bytes(out)


def zero_rle_encode(data: bytes) -> bytes:
    a = np.frombuffer(bytes(data), np.uint8)
    if a.size == 0:
        return b""
    z = np.concatenate(([0], (a == 0).astype(np.int8), [0]))
    edges = np.flatnonzero(np.diff(z))
    runs = [(s, e) for s, e in zip(edges[0::2], edges[1::2]) if e - s >= _MIN_RUN]
    out = bytearray()
    pos = 0

    def lits(lo, hi):
        for o in range(lo, hi, _MAX_LIT):
            part = a[o:min(hi, o + _MAX_LIT)]
            out.append(part.size)
            out.extend(part.tobytes())

    for s, e in runs:
        lits(pos, s)
        out.append(0)
        out += _leb(int(e - s))
        pos = e
    lits(pos, a.size)
    return bytes(out)


def zero_rle_decode(data: bytes) -> bytes:
    data = bytes(data)
    out = bytearray()
    pos, n = 0, len(data)
    while pos < n:
        c = data[pos]
        pos += 1
        if c == 0:
            v = shift = 0
            while True:
                if pos >= n:
                    raise E.CorruptPayload("run length cut short")
                b = data[pos]
                pos += 1
                v |= (b & 0x7F) << shift
                if not b & 0x80:
                    break
                shift += 7
                if shift > 63:
                    raise E.CorruptPayload("run length too wide")
            if v == 0:
                raise E.CorruptPayload("zero-length run")
            out += bytes(v)
        elif c == 0xFF:
            raise E.CorruptPayload("reserved control byte 0xFF")
        else:
            if pos + c > n:
                raise E.CorruptPayload("literal block cut short")
            out += data[pos:pos + c]
            pos += c
    return bytes(out)


_CODECS: dict = {0: (zero_rle_encode, zero_rle_decode)}


def register_secondary_codec(codec_id: int, encode_fn, decode_fn) -> None:
    codec_id = int(codec_id)
    if not 0 <= codec_id <= 255:
        raise ValueError(f"codec_id must fit a byte, got {codec_id}")
    _CODECS[codec_id] = (encode_fn, decode_fn)


def secondary_encode(segment: bytes, codec_id: int = 0) -> bytes:
    if codec_id not in _CODECS:
        raise E.UnknownCodec(f"codec id {codec_id}")
    return bytes([codec_id]) + _CODECS[codec_id][0](bytes(segment))


def secondary_decode(wrapped: bytes) -> bytes:
    if len(wrapped) < 1:
        raise E.CorruptPayload("missing codec id byte")
    cid = wrapped[0]
    if cid not in _CODECS:
        raise E.UnknownCodec(f"codec id {cid}")
    return _CODECS[cid][1](bytes(wrapped[1:]))
