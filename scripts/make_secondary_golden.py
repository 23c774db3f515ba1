"""Golden fixtures for pipelines with a secondary-codec stage:
the REFERENCE fzpipe compresses a few fields through custom pipelines whose
primary segments are wrapped by the zero-RLE secondary codec (pipeline.py:
307-312, encode.py:426-516), and its archives + reconstructions are stored
in tests/golden/secondary.npz.  Needs baseline/_ref (scripts/install_reference.sh).

    python scripts/make_secondary_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/fzpipe_numba_cache")

import fzpipe  # noqa: E402
from fzpipe.data import SyntheticSpec, generate  # noqa: E402
from fzpipe.pipeline import PipelineSpec, StageKind, StageSpec, register_pipeline  # noqa: E402

# (pipeline id, predictor, primary codec)
SPECS = [(60, "lorenzo", "bitshuffle"), (61, "lorenzo", "huffman"), (62, "interp", "huffman")]
FIELDS = [("smooth_trig", (40, 40), 6, 1e-2), ("smooth_trig", (24, 40, 56), 1, 1e-4),
          ("filtered_noise", (64, 64), 3, 1e-3), ("particle1d", (50000,), 2, 1e-4)]


def specs():
    out = []
    for pid, pred, codec in SPECS:
        out.append(PipelineSpec(pid, (
            StageSpec("predict", StageKind.PREDICT, {"predictor": pred}),
            StageSpec("encode", StageKind.PRIMARY_CODEC, {"codec": codec}),
            StageSpec("shrink", StageKind.SECONDARY_CODEC, {"codec_id": "0"}),
        )))
    return out


def main():
    for s in specs():
        register_pipeline(s)
    arr = {"spec_ids": np.array([p for p, _, _ in SPECS]), "spec_pred": np.array([p for _, p, _ in SPECS]),
           "spec_codec": np.array([c for _, _, c in SPECS])}
    names = []
    for kind, dims, seed, rel in FIELDS:
        params = {"width": "2"} if kind == "filtered_noise" else {}
        f = generate(SyntheticSpec(kind, dims, seed, params))
        for pid, _, _ in SPECS:
            name = f"{kind}_{'x'.join(map(str, dims))}_{pid}"
            a = fzpipe.compress(f, fzpipe.ErrorBoundSpec(fzpipe.ErrorMode.VALUE_RANGE_RELATIVE, rel), pid)
            blob = fzpipe.serialize_archive(a)
            r = fzpipe.decompress(fzpipe.parse_archive(blob))
            arr[f"{name}__orig"] = f.data
            arr[f"{name}__dims"] = np.array(dims)
            arr[f"{name}__rel"] = np.array([rel])
            arr[f"{name}__pid"] = np.array([pid])
            arr[f"{name}__archive"] = np.frombuffer(blob, np.uint8)
            arr[f"{name}__recon"] = r.data
            names.append(name)
    arr["names"] = np.array(names)
    out = os.path.join(ROOT, "tests", "golden", "secondary.npz")
    np.savez_compressed(out, **arr)
    print(out, len(names), "archives")


if __name__ == "__main__":
    main()
