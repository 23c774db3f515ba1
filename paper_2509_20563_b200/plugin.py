"""Install the B200 path INTO an unmodified fzpipe (the reference package).

    import fzpipe
    from paper_2509_20563_b200 import plugin
    plugin.install()          # fzpipe's own pipeline now runs the sm_100a kernels
    ...
    plugin.uninstall()

fzpipe's executor reaches its modules through `fzpipe.pipeline`'s imported
predictor names and the `fzpipe.encode` module (pipeline.py:33, 61-67,
269-297, 415-436).  `install` rebinds exactly those names to wrappers that
run this package's GPU implementations and hand back fzpipe's OWN types
(`fzpipe.core.QuantOutput`, `fzpipe.encode.Histogram`,
`fzpipe.encode.HuffmanCodebook`, `fzpipe.core.Field`) and raise fzpipe's OWN
exception classes, so fzpipe's pipeline, container and tests run unchanged
on top.  `calls` counts the GPU calls per entry point (so a test can prove
the kernels, not the numba path, produced the bytes).

Not rebound: the numba kernels fzpipe's task-graph decompress
(pipeline.py:490-580) calls directly, the secondary codec and the metrics.
"""

from __future__ import annotations

import functools
from collections import Counter

calls: Counter = Counter()
_saved: dict = {}


def _translate(fn_name, fzerrors):
    """Map this package's FZError subclasses onto fzpipe's classes of the same name."""
    from . import errors as E

    def deco(f):
        @functools.wraps(f)
        def run(*a, **k):
            calls[fn_name] += 1
            try:
                return f(*a, **k)
            except E.FZError as e:
                cls = getattr(fzerrors, type(e).__name__, None)
                if cls is None or isinstance(e, cls):
                    raise
                if type(e).__name__ == "StageError":
                    raise cls(e.stage, e.cause) from e
                raise cls(str(e)) from e
        return run
    return deco


def install(fzpipe_pkg=None) -> None:
    """Rebind fzpipe's predictor and encoder entry points to the GPU path."""
    if _saved:
        return
    if fzpipe_pkg is None:
        import fzpipe as fzpipe_pkg  # noqa: F401
    import fzpipe.core as RC
    import fzpipe.encode as RE
    import fzpipe.errors as RX
    import fzpipe.pipeline as RP
    import fzpipe.predict as RPR

    from . import encode as ge
    from . import predict as gp

    def quant(q):
        return RC.QuantOutput(q.codes, q.radius, q.outlier_indices, q.outlier_values, q.dims)

    def icfg(cfg):
        return gp.InterpConfig(cfg.anchor_stride, tuple(cfg.cubic_weights))

    def field(f):
        return RC.Field(f.dims, f.data)

    T = lambda name: _translate(name, RX)

    @T("lorenzo_quantize")
    def lorenzo_quantize(fld, bound, radius=512):
        return quant(gp.lorenzo_quantize(fld, bound, radius))

    @T("lorenzo_reconstruct")
    def lorenzo_reconstruct(q, bound):
        return field(gp.lorenzo_reconstruct(q, bound))

    @T("interp_quantize")
    def interp_quantize(fld, bound, radius=512, cfg=RPR.InterpConfig()):
        q, anchors = gp.interp_quantize(fld, bound, radius, icfg(cfg))
        return quant(q), anchors

    @T("interp_reconstruct")
    def interp_reconstruct(q, anchors, bound, cfg=RPR.InterpConfig()):
        return field(gp.interp_reconstruct(q, anchors, bound, icfg(cfg)))

    @T("histogram_exact")
    def histogram_exact(codes, radius):
        h = ge.histogram_exact(codes, radius)
        return RE.Histogram(h.bins, h.total)

    @T("histogram_topk")
    def histogram_topk(codes, radius, k=RE.TOPK_DEFAULT_K):
        h = ge.histogram_topk(codes, radius, k)
        return RE.Histogram(h.bins, h.total)

    @T("huffman_encode")
    def huffman_encode(codes, hist):
        cb, stream, bits = ge.huffman_encode(codes, hist)
        return RE.HuffmanCodebook(cb.code_lengths), stream, bits

    @T("huffman_decode")
    def huffman_decode(cb, bitstream, n):
        return ge.huffman_decode(cb, bitstream, n)

    @T("bitshuffle_encode")
    def bitshuffle_encode(codes, radius):
        return ge.bitshuffle_encode(codes, radius)

    @T("bitshuffle_decode")
    def bitshuffle_decode(bitmap, payload, n, radius):
        return ge.bitshuffle_decode(bitmap, payload, n, radius)

    for mod, name, fn in [(RP, "lorenzo_quantize", lorenzo_quantize), (RP, "lorenzo_reconstruct", lorenzo_reconstruct),
                          (RP, "interp_quantize", interp_quantize), (RP, "interp_reconstruct", interp_reconstruct),
                          (RE, "histogram_exact", histogram_exact), (RE, "histogram_topk", histogram_topk),
                          (RE, "huffman_encode", huffman_encode), (RE, "huffman_decode", huffman_decode),
                          (RE, "bitshuffle_encode", bitshuffle_encode), (RE, "bitshuffle_decode", bitshuffle_decode)]:
        _saved[(mod, name)] = getattr(mod, name)
        setattr(mod, name, fn)


def uninstall() -> None:
    for (mod, name), fn in _saved.items():
        setattr(mod, name, fn)
    _saved.clear()


def installed() -> bool:
    return bool(_saved)


# pytest entry point: `pytest -p paper_2509_20563_b200.plugin <fzpipe tests>`
# runs the reference's own test suite with the GPU path installed.
def pytest_configure(config):  # pragma: no cover - exercised on the GPU box
    install()
