"""CR / PSNR / error statistics with the reference's conventions (fzpipe metrics.py:49-126)."""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import errors as E


@dataclass(frozen=True)
class QualityReport:
    max_abs_err: float
    mse: float
    psnr_db: float
    nrmse: float
    bound_satisfied: bool


@dataclass(frozen=True)
class RateReport:
    cr: float
    bitrate_bits_per_value: float
    input_bytes: int
    compressed_bytes: int


def quality_arrays(orig: np.ndarray, recon: np.ndarray, eb_abs: float | None = None) -> QualityReport:
    o = orig.astype(np.float64)
    d = o - recon.astype(np.float64)
    max_err = float(np.abs(d).max()) if d.size else 0.0
    mse = float(np.mean(d * d)) if d.size else 0.0
    rng = float(o.max() - o.min()) if d.size else 0.0
    if mse == 0.0:
        psnr, nrmse = math.inf, 0.0
    elif rng == 0.0:
        psnr, nrmse = -math.inf, math.inf
    else:
        psnr = 20.0 * math.log10(rng) - 10.0 * math.log10(mse)
        nrmse = math.sqrt(mse) / rng
    return QualityReport(max_err, mse, psnr, nrmse, True if eb_abs is None else max_err <= eb_abs)


def quality(orig, recon, eb_abs: float | None = None) -> QualityReport:
    if orig.dims != recon.dims:
        raise E.DimMismatch(f"{orig.dims} vs {recon.dims}")
    return quality_arrays(orig.data, recon.data, eb_abs)


def rate(input_bytes: int, compressed_bytes: int, element_count: int) -> RateReport:
    input_bytes, compressed_bytes, element_count = int(input_bytes), int(compressed_bytes), int(element_count)
    if input_bytes <= 0 or element_count <= 0:
        raise ValueError("input_bytes and element_count must be positive")
    if compressed_bytes <= 0:
        raise E.ZeroCompressedSize("compressed size must be positive")
    cr = input_bytes / compressed_bytes
    br = 32.0 / cr if input_bytes == 4 * element_count else 8.0 * compressed_bytes / element_count
    return RateReport(cr, br, input_bytes, compressed_bytes)


def throughput(bytes_processed: int, wall_seconds: float) -> float:
    if not wall_seconds > 0:
        raise ValueError("wall_seconds must be positive")
    return bytes_processed / 1e9 / wall_seconds
