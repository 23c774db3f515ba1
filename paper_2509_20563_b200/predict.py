"""Predictor-quantizer modules with the reference API (fzpipe predict.py).

lorenzo_quantize / lorenzo_reconstruct and interp_quantize /
interp_reconstruct run the exact sm_100a kernels (csrc/lorenzo.cu,
csrc/interp.cu) and return the reference's types.  Results are bitwise
identical to the reference: same codes, same outlier list, same recon.
"""

from __future__ import annotations

import ctypes
import enum
import logging
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import errors as E
from .core import Field, QuantOutput, ResolvedBound
from .device import CUBIC, _p, default_engine, interp_applicable, pad3

log = logging.getLogger(__name__)


class PredictorKind(enum.Enum):
    LORENZO = "lorenzo"
    INTERP = "interp"


@dataclass(frozen=True)
class InterpConfig:
    anchor_stride: int = 16
    cubic_weights: tuple = CUBIC

    def __post_init__(self):
        a = int(self.anchor_stride)
        if a < 4 or a & (a - 1):
            raise ValueError(f"anchor_stride must be a power of two >= 4, got {a}")
        w = tuple(float(x) for x in self.cubic_weights)
        if len(w) != 4:
            raise ValueError("cubic_weights needs exactly 4 entries")
        if abs(sum(w) - 1.0) > 1e-12:
            raise ValueError(f"cubic_weights must sum to 1, got {sum(w)!r}")
        object.__setattr__(self, "anchor_stride", a)
        object.__setattr__(self, "cubic_weights", w)


def _radius_ok(radius: int):
    if not 1 <= int(radius) <= 32768:
        raise E.RadiusTooLarge(f"radius {radius} outside the device path's 16-bit code range")


def _compact(eng, x, bitmap, n):
    oidx = eng.buf("p_oidx", 8 * n)
    oval = eng.buf("p_oval", 4 * n)
    cnt = eng.buf("p_ocount", 8)
    ws = eng.buf("p_ocws", eng.lib.fzb_outlier_workspace_bytes(n))
    eng._call("fzb_outlier_compact", _p(bitmap), n, _p(x), _p(oidx), _p(oval), _p(cnt), _p(ws), ws.numel(), eng.sp)
    k = int(cnt[:8].cpu().numpy().view(np.uint64)[0])
    idx = oidx[:8 * k].cpu().numpy().view(np.uint64).astype(np.int64)
    vals = oval[:4 * k].cpu().numpy().view(np.float32).copy()
    return idx, vals


def lorenzo_quantize(field: Field, bound: ResolvedBound, radius: int = 512) -> QuantOutput:
    """predict.py:221-239 on the GPU (exact tiled wavefront / 1D event walk)."""
    _radius_ok(radius)
    eng = default_engine()
    n = field.len
    n0, n1, n2 = pad3(field.dims)
    x = eng.upload("p_x", field.data)[: 4 * n].view(torch.float32)
    eb = eng.upload("p_eb", np.array([bound.eb_abs], np.float64))
    codes = eng.buf("p_codes", 2 * n + 16)
    bitmap = eng.buf("p_bitmap", 4 * ((n + 31) // 32), zero=True)
    ws = eng.buf("p_lzws", eng.lib.fzb_lorenzo_workspace_bytes(n0, n1, n2), zero_new=True)
    eng._call("fzb_lorenzo_encode_f32", _p(x), n0, n1, n2, _p(eb), int(radius), _p(codes), _p(bitmap), _p(ws),
              ws.numel(), eng.sp)
    idx, vals = _compact(eng, x, bitmap, n)
    c = codes[: 2 * n].cpu().numpy().view(np.uint16).astype(np.uint32)
    return QuantOutput(c, int(radius), idx, vals, field.dims)


def _reconstruct(q: QuantOutput, bound: ResolvedBound, predictor: str, anchors: bytes, stride: int) -> Field:
    if q.codes.size and int(q.codes.max()) >= 2 * q.radius:
        raise E.MalformedCodes("code >= 2*radius")
    _radius_ok(q.radius)
    eng = default_engine()
    n = q.codes.size
    codes = eng.upload("p_dcodes", q.codes.astype(np.uint16), pad=16)
    eng.buf("dstatus", 8, zero=True)
    rec = eng.reconstruct(predictor, codes, q.outlier_indices.astype(np.uint64), q.outlier_values, anchors, q.dims,
                          bound.eb_abs, q.radius, stride)
    st = eng.decode_status()
    if st & (_lib.ERR_OUTLIER_CODE | _lib.ERR_OUTLIER_ORDER | _lib.ERR_OUTLIER_RANGE):
        raise E.MalformedCodes("inconsistent outliers")
    return Field(q.dims, rec[:n].cpu().numpy())


def lorenzo_reconstruct(q: QuantOutput, bound: ResolvedBound) -> Field:
    """predict.py:242-253 -- bit-exact vs the encoder's reconstruction."""
    return _reconstruct(q, bound, "lorenzo", b"", 16)


def interp_quantize(field: Field, bound: ResolvedBound, radius: int = 512,
                    cfg: InterpConfig = InterpConfig()):
    """predict.py:270-290 -> (QuantOutput, anchor bytes); Lorenzo fallback for 1D / small extents."""
    if not interp_applicable(field.dims, cfg.anchor_stride):
        log.warning("interpolation needs a 2D or 3D field with every extent >= %d, got dims %s; "
                    "falling back to Lorenzo", cfg.anchor_stride + 1, field.dims)
        return lorenzo_quantize(field, bound, radius), b""
    _radius_ok(radius)
    eng = default_engine()
    n = field.len
    n0, n1, n2 = pad3(field.dims)
    a = cfg.anchor_stride
    na = ((n0 - 1) // a + 1) * ((n1 - 1) // a + 1) * ((n2 - 1) // a + 1)
    x = eng.upload("p_x", field.data)[: 4 * n].view(torch.float32)
    eb = eng.upload("p_eb", np.array([bound.eb_abs], np.float64))
    codes = eng.buf("p_codes", 2 * n + 16)
    bitmap = eng.buf("p_bitmap", 4 * ((n + 31) // 32), zero=True)
    recon = eng.buf("p_recon", 4 * n)
    anchors = eng.buf("p_anchors", 4 * na)
    eng._call("fzb_fill_u16", _p(codes), n, int(radius), eng.sp)
    w = (ctypes.c_double * 4)(*cfg.cubic_weights)
    eng._call("fzb_interp_encode_f32", _p(x), n0, n1, n2, _p(eb), int(radius), a, w, _p(codes), _p(recon),
              _p(bitmap), _p(anchors), eng.sp)
    idx, vals = _compact(eng, x, bitmap, n)
    c = codes[: 2 * n].cpu().numpy().view(np.uint16).astype(np.uint32)
    anc = anchors[: 4 * na].cpu().numpy().tobytes()
    return QuantOutput(c, int(radius), idx, vals, field.dims), anc


def interp_reconstruct(q: QuantOutput, anchors: bytes, bound: ResolvedBound,
                       cfg: InterpConfig = InterpConfig()) -> Field:
    """predict.py:322-344 (empty anchors means the Lorenzo fallback)."""
    if len(anchors) == 0:
        return lorenzo_reconstruct(q, bound)
    if q.codes.size and int(q.codes.max()) >= 2 * q.radius:
        raise E.MalformedCodes("code >= 2*radius")
    a = cfg.anchor_stride
    d3 = pad3(q.dims)
    want = 4 * int(np.prod([(d - 1) // a + 1 for d in d3]))
    if len(anchors) != want:
        raise E.AnchorSizeMismatch(f"anchor payload is {len(anchors)} bytes, expected {want}")
    if tuple(cfg.cubic_weights) != tuple(CUBIC):
        raise ValueError("the device interpolation decoder uses the reference cubic weights")
    return _reconstruct(q, bound, "interp", bytes(anchors), a)
