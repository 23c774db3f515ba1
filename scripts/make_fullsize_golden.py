"""Pin full-size BASELINE configs to the REFERENCE: SHA-256 of fzpipe's input
field, archive and reconstruction bytes for C1-C4 (BASELINE.json configs
0-3) on fzpipe.data.generate inputs, written to tests/golden/fullsize.json.

Runs the reference fzpipe (copied to /tmp/fzref, numba cache in /tmp) in
this container -- a few minutes of single-core CPU.  The GPU box never needs
the reference: tests/test_fullsize.py checks the oracle (CPU) and the CUDA
path (GPU) against these hashes.

    python scripts/make_fullsize_golden.py [name ...]
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import _import_fzpipe  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "fullsize.json")

# name -> (generator kind, dims, seed, rel eb, presets)
CASES = {
    "c1": ("smooth_trig", (100, 500, 500), 0, 1e-4, ("default", "speed", "quality")),
    "c2": ("smooth_trig", (512, 512, 512), 0, 1e-3, ("speed", "default")),
    "c3": ("smooth_trig", (1800, 3600), 0, 1e-4, ("quality",)),
    "c4": ("particle1d", (280953867,), 0, 1e-4, ("default", "speed", "quality")),
}


def sha(b) -> str:
    return hashlib.sha256(bytes(b)).hexdigest()


def main():
    fz = _import_fzpipe()
    from fzpipe.data import SyntheticSpec, generate
    from fzpipe.metrics import quality
    res = json.load(open(OUT)) if os.path.exists(OUT) else {}
    names = sys.argv[1:] or list(CASES)
    for name in names:
        kind, dims, seed, rel, presets = CASES[name]
        t0 = time.time()
        f = generate(SyntheticSpec(kind, dims, seed))
        ent = {"kind": kind, "dims": list(dims), "seed": seed, "rel_eb": rel,
               "input_sha256": sha(f.data.tobytes()), "archives": {}}
        eb = fz.ErrorBoundSpec(fz.ErrorMode.VALUE_RANGE_RELATIVE, rel)
        for p in presets:
            a = fz.compress(f, eb, p)
            blob = fz.serialize_archive(a)
            r = fz.decompress(fz.parse_archive(blob))
            q = quality(f, r, a.resolved_bound().eb_abs)
            ent["archives"][p] = {"archive_sha256": sha(blob), "archive_bytes": len(blob),
                                  "recon_sha256": sha(r.data.tobytes()), "cr": 4 * f.len / len(blob),
                                  "psnr_db": q.psnr_db, "max_abs_err": q.max_abs_err,
                                  "outliers": len(a.segment(2) or b"") // 8}
            print(name, p, ent["archives"][p], f"{time.time() - t0:.1f}s", flush=True)
        res[name] = ent
        json.dump(res, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
