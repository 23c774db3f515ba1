"""ctypes binding of libfzb200.so (the C ABI declared in include/fzb200.h).

There is deliberately no CPU fallback: if the library or a CUDA device is
missing, every entry point raises DeviceUnavailable.
"""

from __future__ import annotations

import ctypes
import os

from . import errors as E

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("FZB_SO") or os.path.join(HERE, "libfzb200.so")  # FZB_SO: tuning builds only

# device status bits (csrc/common.cuh)
ERR_CODE_RANGE = 1 << 0
ERR_MALFORMED = 1 << 1
ERR_HF_TRUNCATED = 1 << 2
ERR_HF_CORRUPT = 1 << 3
ERR_HF_LONG = 1 << 4
ERR_HF_PAD = 1 << 5
ERR_BS_PAD = 1 << 6
ERR_BS_RANGE = 1 << 7
ERR_NONFINITE = 1 << 8
ERR_OUTLIER_RANGE = 1 << 9
ERR_OUTLIER_ORDER = 1 << 10
ERR_OUTLIER_CODE = 1 << 11
ERR_HF_MISMATCH = 1 << 12
ERR_HF_SYNC = 1 << 13
ERR_BS_MISMATCH = 1 << 14
ERR_DQ_RANGE = 1 << 15

# (bit, exception factory), in the order the reference would raise them
CODEC_ERRORS = [
    (ERR_HF_TRUNCATED, lambda: E.Truncated("bitstream ended mid-symbol")),
    (ERR_HF_CORRUPT, lambda: E.CorruptStream("bit pattern matches no codeword")),
    (ERR_HF_LONG, lambda: E.CorruptStream("bitstream longer than the decoded symbols need")),
    (ERR_HF_PAD, lambda: E.CorruptStream("nonzero padding bits")),
    (ERR_BS_MISMATCH, lambda: E.BitmapPayloadMismatch("bitmap popcount disagrees with payload words")),
    (ERR_BS_PAD, lambda: E.CorruptPayload("nonzero bits in block padding")),
    (ERR_BS_RANGE, lambda: E.CorruptPayload("decoded code >= 2*radius")),
    (ERR_HF_MISMATCH, lambda: E.CorruptStream("histogram inconsistent with codes")),
    (ERR_CODE_RANGE, lambda: E.CodeOutOfRange("code >= 2*radius")),
]

_lib = None


class LaunchError(RuntimeError):
    pass


def load():
    """Load (and, when missing or stale in a build tree, compile) the library."""

    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO_PATH):
        try:
            from .build import build
            build()
        except Exception as e:  # no nvcc / failed build
            raise E.DeviceUnavailable(f"libfzb200.so missing and could not be built: {e}") from e
    L = ctypes.CDLL(SO_PATH)
    P, U32, U64, I, D, SZ = (ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_double,
                             ctypes.c_size_t)
    sig = {
        "fzb_abi_version": (I, []),
        "fzb_event_create": (I, [P]),
        "fzb_event_destroy": (I, [P]),
        "fzb_event_record": (I, [P, P, I]),
        "fzb_event_elapsed_ms": (I, [P, P, P]),
        "fzb_minmax_workspace_bytes": (SZ, [U64]),
        "fzb_minmax_f32": (I, [P, U64, P, P, SZ, P, P]),
        "fzb_resolve_bound": (I, [P, I, D, P, P]),
        "fzb_lorenzo_workspace_bytes": (SZ, [U32, U32, U32]),
        "fzb_lorenzo_encode_f32": (I, [P, U32, U32, U32, P, U32, P, P, P, SZ, P]),
        "fzb_lorenzo_decode_f32": (I, [P, P, P, U32, U32, U32, P, U32, P, SZ, P]),
        "fzb_lorenzo_batch_workspace_bytes": (SZ, [U32, U32, U32, U32]),
        "fzb_lorenzo_encode_batch_f32": (I, [P, U32, U64, U32, U32, U32, P, U32, P, P, U64, P, SZ, P]),
        "fzb_lorenzo_decode_batch_f32": (I, [P, P, U64, P, U32, U64, U32, U32, U32, P, U32, P, SZ, P]),
        "fzb_interp_encode_f32": (I, [P, U32, U32, U32, P, U32, U32, P, P, P, P, P, P]),
        "fzb_interp_decode_f32": (I, [P, P, P, P, U32, U32, U32, P, U32, U32, P, P]),
        "fzb_outlier_workspace_bytes": (SZ, [U64]),
        "fzb_outlier_compact": (I, [P, U64, P, P, P, P, P, SZ, P]),
        "fzb_outlier_scatter": (I, [P, P, U64, U64, P, U32, P, P, P, P]),
        "fzb_outlier_check": (I, [P, U64, U64, P, U32, P, P]),
        "fzb_quality_leaves": (I, [P, P, P, P, U64, P, P, P]),
        "fzb_histogram": (I, [P, U64, U32, P, P, P]),
        "fzb_lorenzo1d_prepare_f32": (I, [P, U64, U32, P, P, P, SZ, P, P]),
        "fzb_lorenzo1d_walk_f32": (I, [P, U64, P, U32, P, P, P, P, SZ, P]),
        "fzb_histogram_flagged": (I, [P, U64, U32, P, P, P, P]),
        "fzb_histogram_chunks": (I, [P, U64, U32, P, P, P, P]),
        "fzb_huffman_build_workspace_bytes": (SZ, [U32]),
        "fzb_huffman_build": (I, [P, U32, P, P, P, P, SZ, P]),
        "fzb_huffman_encode_workspace_bytes": (SZ, [U64]),
        "fzb_huffman_encode": (I, [P, U64, P, P, U32, P, P, U64, P, SZ, P, P]),
        "fzb_huffman_encode_chunks": (I, [P, U64, P, P, U32, P, P, P, U64, P, SZ, P, P]),
        "fzb_huffman_decode_workspace_bytes": (SZ, [U64, U32]),
        "fzb_huffman_decode": (I, [P, U64, U64, P, U32, P, P, SZ, P, P]),
        "fzb_bitshuffle_workspace_bytes": (SZ, [U64]),
        "fzb_bitshuffle_encode": (I, [P, U64, P, P, P, P, SZ, P]),
        "fzb_bitshuffle_decode": (I, [P, P, U64, U64, U32, P, P, SZ, P, P]),
        "fzb_fill_u16": (I, [P, U64, ctypes.c_uint16, P]),
        "fzb_interp_profile": (I, [P, U32, U32, U32, P, P, P]),
        "fzb_dualquant_encode_f32": (I, [P, U32, U32, U32, P, U32, P, P, P, P]),
        "fzb_dualquant_outlier_deltas": (I, [P, U32, U32, U32, P, P, P, U32, P, P, P]),
        "fzb_dualquant_decode_workspace_bytes": (SZ, [U32, U32, U32]),
        "fzb_dualquant_decode_f32": (I, [P, P, P, P, U64, U32, U32, U32, P, U32, P, P, P, SZ, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


EXPORTED = [
    "fzb_abi_version", "fzb_event_create", "fzb_event_destroy", "fzb_event_record", "fzb_event_elapsed_ms", "fzb_minmax_workspace_bytes", "fzb_minmax_f32", "fzb_resolve_bound",
    "fzb_lorenzo_workspace_bytes", "fzb_lorenzo_encode_f32", "fzb_lorenzo_decode_f32",
    "fzb_lorenzo_batch_workspace_bytes", "fzb_lorenzo_encode_batch_f32", "fzb_lorenzo_decode_batch_f32",
    "fzb_interp_encode_f32",
    "fzb_interp_decode_f32", "fzb_outlier_workspace_bytes", "fzb_outlier_compact", "fzb_outlier_scatter",
    "fzb_outlier_check",
    "fzb_quality_leaves",
    "fzb_histogram", "fzb_histogram_chunks", "fzb_lorenzo1d_prepare_f32", "fzb_lorenzo1d_walk_f32",
    "fzb_histogram_flagged", "fzb_huffman_encode_chunks", "fzb_huffman_build_workspace_bytes", "fzb_huffman_build", "fzb_huffman_encode_workspace_bytes",
    "fzb_huffman_encode", "fzb_huffman_decode_workspace_bytes", "fzb_huffman_decode",
    "fzb_bitshuffle_workspace_bytes", "fzb_bitshuffle_encode", "fzb_bitshuffle_decode", "fzb_fill_u16",
    "fzb_interp_profile", "fzb_dualquant_encode_f32", "fzb_dualquant_outlier_deltas", "fzb_dualquant_decode_workspace_bytes",
    "fzb_dualquant_decode_f32",
]


def check(rc: int, what: str) -> None:
    if rc == -1002:
        raise E.RadiusTooLarge(f"{what}: radius outside [1, 32768]")
    if rc != 0:
        raise LaunchError(f"{what} failed with status {rc}")


def raise_codec_status(bits: int) -> None:
    """Raise the reference exception for data-dependent codec failures."""

    for bit, make in CODEC_ERRORS:
        if bits & bit:
            raise make()
