"""Synthetic SDRBench-shaped fields (counter-based SplitMix64), host and device.

Same generator definitions as the reference's data.py (smooth_trig,
particle1d, filtered_noise without the scipy filter); the device variant
runs the f64 math on the GPU so a 512^3 field takes milliseconds instead of
~18 s of numpy.  Bench inputs only need to be "SDRBench-shaped"; parity is
always checked on the exact bytes the GPU consumed.
"""

from __future__ import annotations

import math

import numpy as np
import torch

GAMMA = 0x9E3779B97F4A7C15
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB
MASK = (1 << 64) - 1


def splitmix_uniform_host(seed: int, start: int, count: int) -> np.ndarray:
    i = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    z = i * np.uint64(GAMMA) + np.uint64(seed & MASK)
    z ^= z >> np.uint64(30)
    z *= np.uint64(M1)
    z ^= z >> np.uint64(27)
    z *= np.uint64(M2)
    z ^= z >> np.uint64(31)
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def _to_i64(v: int) -> int:
    v &= MASK
    return v - (1 << 64) if v >> 63 else v


def splitmix_uniform_device(seed: int, start: int, count: int, device) -> torch.Tensor:
    """int64 two's-complement arithmetic == uint64 mod 2^64; logical shifts masked."""
    i = torch.arange(start + 1, start + count + 1, dtype=torch.int64, device=device)
    z = i * _to_i64(GAMMA) + _to_i64(seed)

    def lsr(x, k):
        return (x >> k) & ((1 << (64 - k)) - 1)

    z = z ^ lsr(z, 30)
    z = z * _to_i64(M1)
    z = z ^ lsr(z, 27)
    z = z * _to_i64(M2)
    z = z ^ lsr(z, 31)
    return lsr(z, 11).to(torch.float64) * 2.0 ** -53


def _trig_terms(dims, seed, terms=4, max_cycles=2.0):
    nd = len(dims)
    draws = splitmix_uniform_host(seed, 0, terms * (nd + 2))
    out = []
    for t in range(terms):
        d0 = t * (nd + 2)
        freqs = 0.25 + (max_cycles - 0.25) * draws[d0:d0 + nd]
        out.append((freqs, 2.0 * math.pi * draws[d0 + nd], (0.5 + draws[d0 + nd + 1]) / (t + 1)))
    return out


def smooth_trig_host(dims, seed: int = 0) -> np.ndarray:
    """fzpipe data._smooth_trig (data.py:85-106) bit for bit: the same per-
    element operation order, evaluated in slabs of the slowest axis to bound
    the f64 temporaries (every element's arithmetic is independent)."""
    dims = tuple(int(d) for d in dims)
    coords = [np.arange(d, dtype=np.float64) / d for d in dims]
    terms = _trig_terms(dims, seed)
    out = np.empty(dims, np.float32)
    per = int(np.prod(dims[1:])) if len(dims) > 1 else 1
    step = max(1, (1 << 22) // per)
    for s0 in range(0, dims[0], step):
        s1 = min(dims[0], s0 + step)
        shp = (s1 - s0,) + dims[1:]
        acc = np.zeros(shp, np.float64)
        for freqs, phase, amp in terms:
            arg = np.full(shp, phase)
            for ax, d in enumerate(dims):
                shape = [1] * len(dims)
                shape[ax] = shp[ax]
                c = coords[ax][s0:s1] if ax == 0 else coords[ax]
                arg = arg + (2.0 * np.pi * freqs[ax] * c).reshape(shape)
            acc += amp * np.sin(arg)
        out[s0:s1] = acc.astype(np.float32)
    return out.reshape(-1)


def smooth_trig_device(dims, seed: int = 0, device="cuda") -> torch.Tensor:
    """f32 field on the device; chunks the slowest axis to bound f64 temporaries."""
    dims = tuple(int(d) for d in dims)
    out = torch.empty(int(np.prod(dims)), dtype=torch.float32, device=device)
    terms = _trig_terms(dims, seed)
    lead = dims[0]
    rest = dims[1:]
    per = int(np.prod(rest)) if rest else 1
    step = max(1, (1 << 25) // max(per, 1))
    axes = [torch.arange(d, dtype=torch.float64, device=device) / d for d in dims]
    for s0 in range(0, lead, step):
        s1 = min(lead, s0 + step)
        shp = (s1 - s0,) + rest
        acc = torch.zeros(shp, dtype=torch.float64, device=device)
        for freqs, phase, amp in terms:
            arg = torch.full(shp, phase, dtype=torch.float64, device=device)
            for ax in range(len(dims)):
                v = 2.0 * math.pi * float(freqs[ax]) * (axes[ax][s0:s1] if ax == 0 else axes[ax])
                view = [1] * len(dims)
                view[ax] = v.numel()
                arg = arg + v.reshape(view)
            acc += amp * torch.sin(arg)
        out[s0 * per:s1 * per] = acc.reshape(-1).to(torch.float32)
    return out


def particle1d_host(n: int, seed: int = 0, box: float = 1000.0, jitter: float = 0.3) -> np.ndarray:
    """fzpipe data._particle1d (data.py:137-147) bit for bit, in chunks."""
    out = np.empty(n, np.float32)
    step = 1 << 22
    for s0 in range(0, n, step):
        s1 = min(n, s0 + step)
        u = splitmix_uniform_host(seed, s0, s1 - s0)
        out[s0:s1] = box * (np.arange(s0, s1, dtype=np.float64) + 0.5 + jitter * (2.0 * u - 1.0)) / n
    return out


def particle1d_device(n: int, seed: int = 0, box: float = 1000.0, jitter: float = 0.3, device="cuda"):
    out = torch.empty(n, dtype=torch.float32, device=device)
    step = 1 << 26
    for s0 in range(0, n, step):
        s1 = min(n, s0 + step)
        u = splitmix_uniform_device(seed, s0, s1 - s0, device)
        i = torch.arange(s0, s1, dtype=torch.float64, device=device)
        out[s0:s1] = (box * (i + 0.5 + jitter * (2.0 * u - 1.0)) / n).to(torch.float32)
    return out


def noise_host(n: int, seed: int = 0) -> np.ndarray:
    return splitmix_uniform_host(seed, 0, n).astype(np.float32)
