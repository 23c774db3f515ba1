"""CR / PSNR / error statistics with the reference's conventions (fzpipe metrics.py:49-126)."""

from __future__ import annotations

import functools
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


@functools.lru_cache(maxsize=8)
def _pairwise_tree(n: int):
    """numpy's pairwise-sum split tree for a contiguous array of n f64
    (numpy loops_utils pairwise_sum: halve at a multiple of 8 until a block
    holds <= 128 values).  Returns the leaves (offset, length) and per level
    the leaf mask, leaf ids and whether the level has children below."""
    sizes = np.array([n], np.int64)
    offs = np.array([0], np.int64)
    levels, leaf_off, leaf_len = [], [], []
    nleaf = 0
    while sizes.size:
        split = sizes > 128
        leaf = ~split
        ids = np.arange(nleaf, nleaf + int(leaf.sum()), dtype=np.int64)
        leaf_off.append(offs[leaf])
        leaf_len.append(sizes[leaf])
        nleaf += ids.size
        levels.append((leaf, ids))
        h = sizes[split] // 2
        h -= h % 8
        m = sizes[split]
        o = offs[split]
        sizes = np.stack([h, m - h], 1).reshape(-1)
        offs = np.stack([o, o + h], 1).reshape(-1)
    return (np.concatenate(leaf_off).astype(np.uint64), np.concatenate(leaf_len).astype(np.uint16), levels)


def quality_device(orig, recon, dims, eb_abs: float | None = None) -> QualityReport:
    """metrics.quality on device-resident f32 tensors (fzpipe metrics.py:49-75),
    bit-identical to the host version: max|d| and the range are exact
    reductions, the MSE follows numpy's pairwise summation tree exactly
    (leaves summed by fzb_quality_leaves, folded up the tree in f64)."""
    import torch
    from .device import _p, default_engine
    n = int(orig.numel())
    if tuple(dims) and int(np.prod(dims)) != n or recon.numel() != n:
        raise E.DimMismatch(f"{n} vs {recon.numel()}")
    if n == 0:
        return QualityReport(0.0, 0.0, math.inf, 0.0, True)
    eng = default_engine()
    off, ln, levels = _pairwise_tree(n)
    dev = orig.device
    d_off = torch.from_numpy(off.view(np.int64)).to(dev)
    d_len = torch.from_numpy(ln.view(np.int16)).to(dev)
    leaf_sum = torch.empty(off.size, dtype=torch.float64, device=dev)
    red = torch.tensor([0, -1, 0], dtype=torch.int64, device=dev)
    eng._call("fzb_quality_leaves", _p(orig), _p(recon), _p(d_off), _p(d_len), off.size, _p(leaf_sum), _p(red),
              eng.sp)
    below = None   # values of the level underneath (children of its split nodes, in order)
    for leaf, ids in reversed(levels):
        vals = torch.empty(leaf.size, dtype=torch.float64, device=dev)
        lm = torch.from_numpy(leaf).to(dev)
        vals[lm] = leaf_sum[torch.from_numpy(ids).to(dev)]
        if below is not None:
            vals[~lm] = below[0::2] + below[1::2]
        below = vals
    total = float(below[0].item())
    r = red.cpu().numpy().view(np.uint64)
    max_err = float(np.array([r[0]], np.uint64).view(np.float64)[0])

    def unkey(k):
        u = np.uint32(k)
        u = np.uint32(u & 0x7FFFFFFF) if u & 0x80000000 else np.uint32(~u)
        return float(np.array([u], np.uint32).view(np.float32)[0])

    mse = total / n
    rng = float(np.float64(unkey(int(r[2]))) - np.float64(unkey(int(r[1]))))
    if mse == 0.0:
        psnr, nrmse = math.inf, 0.0
    elif rng == 0.0:
        psnr, nrmse = -math.inf, math.inf
    else:
        psnr = 20.0 * math.log10(rng) - 10.0 * math.log10(mse)
        nrmse = math.sqrt(mse) / rng
    return QualityReport(max_err, mse, psnr, nrmse, True if eb_abs is None else max_err <= eb_abs)


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
