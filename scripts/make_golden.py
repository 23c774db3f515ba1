"""Generate tests/golden/*.npz by running the REFERENCE fzpipe in this container.

The reference (/root/reference/pkg) is copied to /tmp/fzref so numba's
cache=True does not write next to the read-only sources.  The fixtures
pin the CPU oracle (oracle/fzoracle.py) and, through it, the GPU kernels.
They are small enough to commit; the GPU box never needs the reference.

    python scripts/make_golden.py
"""

from __future__ import annotations

import os
import shutil
import sys

import numpy as np

REF = "/root/reference/pkg"
COPY = "/tmp/fzref"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def _import_fzpipe():
    if not os.path.isdir(COPY):
        shutil.copytree(REF, COPY)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/fzref_numba_cache")
    sys.path.insert(0, os.path.join(COPY, "src"))
    import fzpipe  # noqa: F401
    return fzpipe


def _field(fz, kind, dims, seed, **params):
    from fzpipe.data import SyntheticSpec, generate
    if kind == "uniform":
        rng = np.random.default_rng(seed)
        lo, hi = params.get("lo", -1.0), params.get("hi", 1.0)
        return fz.Field(tuple(dims), rng.uniform(lo, hi, int(np.prod(dims))).astype(np.float32))
    if kind == "array":
        return fz.Field(tuple(dims), np.asarray(params["data"], np.float32))
    p = {k: str(v) for k, v in params.items()}
    return generate(SyntheticSpec(kind, tuple(dims), seed, p))


# (name, field spec, eb mode ('abs'|'rel'), magnitude, radius)
PREDICT_CASES = [
    ("ramp_kat", ("array", (3,), 0, dict(data=[0.0, 1.0, 2.0])), "abs", 0.5, 512),
    ("outlier_kat", ("array", (2,), 0, dict(data=[0.0, 1e6])), "abs", 0.5, 512),
    ("negzero", ("array", (2, 5), 0, dict(data=[-0.0, 0.0, -0.0, 1.0, -0.0, 0.0, 0.0, -0.0, 2.0, -0.0])), "abs", 0.25, 512),
    ("smooth1d", ("smooth_trig", (1000,), 3, {}), "rel", 1e-3, 512),
    ("particle1d", ("particle1d", (50000,), 0, {}), "rel", 1e-4, 512),
    ("noise1d", ("filtered_noise", (5000,), 1, dict(width=2)), "rel", 1e-4, 512),
    ("smooth2d", ("smooth_trig", (33, 41), 2, {}), "rel", 1e-3, 512),
    ("smooth2d_wide", ("smooth_trig", (70, 300), 5, {}), "rel", 1e-4, 512),
    ("smooth2d_tall", ("smooth_trig", (300, 70), 6, {}), "rel", 1e-4, 512),
    ("smooth3d_small", ("smooth_trig", (7, 9, 11), 3, {}), "rel", 1e-3, 512),
    ("smooth3d", ("smooth_trig", (17, 18, 19), 3, {}), "rel", 1e-4, 512),
    ("smooth3d_tiles", ("smooth_trig", (20, 70, 45), 7, {}), "rel", 1e-4, 512),
    ("smooth3d_interp", ("smooth_trig", (40, 33, 21), 11, {}), "rel", 1e-3, 512),
    ("noise3d", ("filtered_noise", (18, 19, 20), 57, dict(width=2)), "rel", 1e-4, 512),
    ("noise2d", ("filtered_noise", (65, 33), 98, dict(width=2)), "abs", 1e-2, 512),
    ("uniform_radius4", ("uniform", (300,), 5, dict(lo=-50.0, hi=50.0)), "abs", 1e-3, 4),
    ("uniform3d_r16", ("uniform", (9, 20, 33), 8, dict(lo=-4.0, hi=4.0)), "abs", 1e-2, 16),
    ("piecewise2d", ("piecewise_constant", (48, 48), 4, dict(block=8)), "rel", 1e-3, 512),
    ("bilinear", ("array", (65, 65), 0, {}), "abs", 1e-4, 512),
]

ARCHIVE_CASES = [
    ("smooth1d", ("smooth_trig", (500,), 1, {}), "rel", 1e-3),
    ("smooth2d", ("smooth_trig", (33, 41), 2, {}), "rel", 1e-3),
    ("smooth3d", ("smooth_trig", (17, 18, 19), 3, {}), "rel", 1e-3),
    ("smooth3d_e4", ("smooth_trig", (24, 40, 56), 9, {}), "rel", 1e-4),
    ("uniform2d_abs", ("uniform", (64, 64), 9, dict(lo=-100.0, hi=100.0)), "abs", 1e-4),
    ("noise3d", ("filtered_noise", (20, 20, 20), 3, dict(width=3)), "rel", 1e-5),
    ("particle1d", ("particle1d", (30000,), 2, {}), "rel", 1e-4),
    ("constant", ("array", (4, 5), 0, dict(data=[1.5] * 20)), "rel", 1e-3),
]


def _bilinear():
    y, x = np.mgrid[0:65, 0:65].astype(np.float64)
    return (0.25 * x + 0.5 * y).astype(np.float32).reshape(-1)


def predict_fixtures(fz):
    from fzpipe.core import ErrorBoundSpec, ErrorMode, resolve_bound
    from fzpipe.predict import InterpConfig, _interp_quantize_with_recon, _lorenzo_quantize_with_recon, _interp_applicable
    out = {}
    for name, (kind, dims, seed, params), mode, mag, radius in PREDICT_CASES:
        if name == "bilinear":
            params = dict(data=_bilinear())
            kind = "array"
        f = _field(fz, kind, dims, seed, **params)
        em = ErrorMode.ABSOLUTE if mode == "abs" else ErrorMode.VALUE_RANGE_RELATIVE
        b = resolve_bound(f, ErrorBoundSpec(em, mag))
        q, rec = _lorenzo_quantize_with_recon(f, b, radius)
        pre = f"{name}__"
        out[pre + "orig"] = f.data
        out[pre + "dims"] = np.array(f.dims, np.int64)
        out[pre + "eb"] = np.array([b.eb_abs], np.float64)
        out[pre + "radius"] = np.array([radius], np.int64)
        out[pre + "lz_codes"] = q.codes.astype(np.uint32)
        out[pre + "lz_oidx"] = q.outlier_indices
        out[pre + "lz_oval"] = q.outlier_values
        out[pre + "lz_recon"] = rec
        if _interp_applicable(f, InterpConfig()):
            qi, reci, anchors = _interp_quantize_with_recon(f, b, radius, InterpConfig())
            out[pre + "ip_codes"] = qi.codes.astype(np.uint32)
            out[pre + "ip_oidx"] = qi.outlier_indices
            out[pre + "ip_oval"] = qi.outlier_values
            out[pre + "ip_recon"] = reci
            out[pre + "ip_anchors"] = np.frombuffer(anchors, np.uint8)
    out["names"] = np.array([c[0] for c in PREDICT_CASES])
    return out


def archive_fixtures(fz):
    from fzpipe.core import ErrorBoundSpec, ErrorMode, serialize_archive
    from fzpipe.pipeline import compress, decompress
    out = {}
    names = []
    for name, (kind, dims, seed, params), mode, mag in ARCHIVE_CASES:
        f = _field(fz, kind, dims, seed, **params)
        em = ErrorMode.ABSOLUTE if mode == "abs" else ErrorMode.VALUE_RANGE_RELATIVE
        out[f"{name}__orig"] = f.data
        out[f"{name}__dims"] = np.array(f.dims, np.int64)
        out[f"{name}__mode"] = np.array([int(em)], np.int64)
        out[f"{name}__mag"] = np.array([mag], np.float64)
        for preset in ("default", "speed", "quality"):
            a = compress(f, ErrorBoundSpec(em, mag), preset)
            blob = serialize_archive(a)
            out[f"{name}__{preset}__archive"] = np.frombuffer(blob, np.uint8)
            out[f"{name}__{preset}__recon"] = decompress(a).data
        names.append(name)
    out["names"] = np.array(names)
    return out


def codebook_fixtures(fz):
    from fzpipe.encode import _package_merge_lengths
    rng = np.random.default_rng(20250920)
    hists, lens, sizes = [], [], []
    for t in range(400):
        nsym = int(rng.choice([2, 3, 4, 8, 16, 64, 256, 1024]))
        h = np.zeros(nsym, np.uint64)
        style = t % 4
        m = int(rng.integers(1, nsym + 1))
        syms = rng.choice(nsym, m, replace=False)
        if style == 0:
            h[syms] = rng.integers(1, 1 << 20, m)
        elif style == 1:  # tie heavy
            h[syms] = rng.integers(1, 4, m)
        elif style == 2:  # geometric: forces the 32-bit length limit
            h[syms] = (np.uint64(1) << np.minimum(np.arange(m), 62).astype(np.uint64))
        else:  # peaked like quant codes
            h[syms] = rng.integers(1, 50, m)
            h[syms[0]] = 10_000_000
        hists.append(h)
        lens.append(_package_merge_lengths(h, 32))
        sizes.append(nsym)
    return dict(hist=np.concatenate(hists), lengths=np.concatenate(lens), sizes=np.array(sizes, np.int64))


def main():
    fz = _import_fzpipe()
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, "predict.npz"), **predict_fixtures(fz))
    np.savez_compressed(os.path.join(OUT, "archives.npz"), **archive_fixtures(fz))
    np.savez_compressed(os.path.join(OUT, "codebooks.npz"), **codebook_fixtures(fz))
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
