"""Pipeline registry and executor -- drop-in for fzpipe.pipeline on the B200.

Same public surface as the reference (pipeline.py:70-660): StageKind,
StageSpec, PipelineSpec (validation + histogram auto-insert), the preset
registry (0 default = Lorenzo + exact histogram + Huffman, 1 speed =
Lorenzo + bitshuffle, 2 quality = interp + top-k histogram + Huffman),
ini pipeline files, compress/decompress (+ _with_timing, _via_graph).
The stage bodies run on the GPU through device.Engine; archives are
byte-identical to the reference's for the same input and spec.
"""

from __future__ import annotations

import configparser
import enum
import logging
import os
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import errors as E
from . import secondary
from .core import (
    SEG_ANCHOR_GRID, SEG_BITSHUFFLE_BITMAP, SEG_BITSHUFFLE_PAYLOAD, SEG_DQ_DELTAS, SEG_HUFFMAN_BITSTREAM,
    SEG_HUFFMAN_CODEBOOK, SEG_INTERP_PROFILE, SEG_OUTLIER_INDICES, SEG_OUTLIER_VALUES, SEG_SECONDARY_WRAPPED, Archive, ErrorBoundSpec,
    ErrorMode, Field,
    ResolvedBound, attach_wire, eb_from_range, register_known_pipeline_id,
)
from .device import default_engine, graph_engine, interp_applicable

log = logging.getLogger(__name__)


class StageKind(enum.Enum):
    PREPROCESS = "preprocess"
    PREDICT = "predict"
    PRIMARY_CODEC = "primary_codec"
    SECONDARY_CODEC = "secondary_codec"
    ANALYSIS = "analysis"


_RANK = {StageKind.PREPROCESS: 0, StageKind.PREDICT: 1, StageKind.ANALYSIS: 2, StageKind.PRIMARY_CODEC: 3,
         StageKind.SECONDARY_CODEC: 4}


@dataclass(frozen=True)
class StageSpec:
    name: str
    kind: StageKind
    params: tuple = ()

    def __post_init__(self):
        if not self.name:
            raise E.InvalidStageOrder("stage name must be nonempty")
        p = self.params
        if isinstance(p, dict):
            p = tuple(sorted((str(k), str(v)) for k, v in p.items()))
        object.__setattr__(self, "params", tuple(p))
        object.__setattr__(self, "kind", StageKind(self.kind))

    def param(self, key: str, default=None):
        return dict(self.params).get(key, default)


@dataclass(frozen=True)
class PipelineSpec:
    id: int
    stages: tuple

    def __post_init__(self):
        pid = int(self.id)
        if not 0 <= pid <= 255:
            raise E.InvalidStageOrder(f"pipeline id must fit a byte, got {pid}")
        stages = tuple(self.stages)
        names = [s.name for s in stages]
        if len(names) != len(set(names)):
            raise E.InvalidStageOrder(f"duplicate stage names in {names}")
        ranks = [_RANK[s.kind] for s in stages]
        if ranks != sorted(ranks):
            raise E.InvalidStageOrder(
                "stage order must be preprocess, predict, analysis, primary codec, secondary codec")
        kinds = [s.kind for s in stages]
        if kinds.count(StageKind.PREDICT) != 1:
            raise E.MissingStage("exactly one predict stage required")
        if kinds.count(StageKind.PRIMARY_CODEC) != 1:
            raise E.MissingStage("exactly one primary codec stage required")
        if kinds.count(StageKind.SECONDARY_CODEC) > 1:
            raise E.InvalidStageOrder("at most one secondary codec stage")
        primary = next(s for s in stages if s.kind == StageKind.PRIMARY_CODEC)
        if primary.param("codec", "huffman") == "huffman" and StageKind.ANALYSIS not in kinds:
            i = stages.index(primary)
            stages = stages[:i] + (StageSpec("histogram", StageKind.ANALYSIS, {"method": "exact"}),) + stages[i:]
        object.__setattr__(self, "id", pid)
        object.__setattr__(self, "stages", stages)

    def stage_of(self, kind: StageKind):
        return next((s for s in self.stages if s.kind == kind), None)

    @property
    def predictor(self) -> str:
        return self.stage_of(StageKind.PREDICT).param("predictor", "lorenzo")

    @property
    def primary_codec(self) -> str:
        return self.stage_of(StageKind.PRIMARY_CODEC).param("codec", "huffman")

    def radius(self) -> int:
        return int(self.stage_of(StageKind.PREDICT).param("radius", "512"))

    def interp_config(self):
        from .predict import InterpConfig
        return InterpConfig(anchor_stride=int(self.stage_of(StageKind.PREDICT).param("anchor_stride", "16")))


_REGISTRY: dict[int, PipelineSpec] = {}
PRESET_NAMES = {"default": 0, "speed": 1, "quality": 2, "dq-speed": 3, "dq-default": 4, "q-profiled": 5}


def register_pipeline(spec: PipelineSpec) -> PipelineSpec:
    if spec.id in _REGISTRY:
        raise E.DuplicateId(f"pipeline id {spec.id} already registered")
    _REGISTRY[spec.id] = spec
    register_known_pipeline_id(spec.id)
    return spec


def get_pipeline(ref) -> PipelineSpec:
    if isinstance(ref, PipelineSpec):
        return ref
    if isinstance(ref, str):
        if ref not in PRESET_NAMES:
            raise E.UnknownPipelineId(f"unknown pipeline name '{ref}'")
        ref = PRESET_NAMES[ref]
    ref = int(ref)
    if ref not in _REGISTRY:
        raise E.UnknownPipelineId(f"pipeline id {ref} not registered")
    return _REGISTRY[ref]


def registered_pipelines() -> dict:
    return dict(_REGISTRY)


def _presets():
    S, K = StageSpec, StageKind
    register_pipeline(PipelineSpec(0, (S("predict", K.PREDICT, {"predictor": "lorenzo"}),
                                       S("histogram", K.ANALYSIS, {"method": "exact"}),
                                       S("encode", K.PRIMARY_CODEC, {"codec": "huffman"}))))
    register_pipeline(PipelineSpec(1, (S("predict", K.PREDICT, {"predictor": "lorenzo"}),
                                       S("encode", K.PRIMARY_CODEC, {"codec": "bitshuffle"}))))
    register_pipeline(PipelineSpec(2, (S("predict", K.PREDICT, {"predictor": "interp"}),
                                       S("histogram", K.ANALYSIS, {"method": "topk", "k": "16"}),
                                       S("encode", K.PRIMARY_CODEC, {"codec": "huffman"}))))
    # opt-in, this repo's own (no reference counterpart): dual-quant Lorenzo
    # (north_star items 1 and 4; csrc/dualquant.cu), with bitshuffle / Huffman
    register_pipeline(PipelineSpec(3, (S("predict", K.PREDICT, {"predictor": "dualquant"}),
                                       S("encode", K.PRIMARY_CODEC, {"codec": "bitshuffle"}))))
    register_pipeline(PipelineSpec(4, (S("predict", K.PREDICT, {"predictor": "dualquant"}),
                                       S("histogram", K.ANALYSIS, {"method": "exact"}),
                                       S("encode", K.PRIMARY_CODEC, {"codec": "huffman"}))))
    # opt-in: G-Interp whose anchor stride (16 | 8) and interpolation weights
    # (cubic | linear | natural cubic) are chosen per field by sampled
    # profiling (cuSZ-i / QoZ; north_star item 2; csrc/interp.cu)
    register_pipeline(PipelineSpec(5, (S("predict", K.PREDICT, {"predictor": "interp", "profile": "1"}),
                                       S("histogram", K.ANALYSIS, {"method": "topk", "k": "16"}),
                                       S("encode", K.PRIMARY_CODEC, {"codec": "huffman"}))))


_presets()


def load_pipeline_file(path: str) -> PipelineSpec:
    """[pipeline] id = N, then one [stage:<name>] section per stage (kind = ...)."""

    cp = configparser.ConfigParser()
    if not cp.read(path):
        raise E.BadParams(f"cannot read pipeline file '{path}'")
    if "pipeline" not in cp or "id" not in cp["pipeline"]:
        raise E.BadParams("pipeline file needs a [pipeline] section with an id")
    try:
        pid = int(cp["pipeline"]["id"])
    except ValueError as e:
        raise E.BadParams(f"bad pipeline id: {e}") from None
    stages = []
    for sec in cp.sections():
        if not sec.startswith("stage:"):
            continue
        opts = dict(cp[sec])
        kind = opts.pop("kind", None)
        if kind is None:
            raise E.BadParams(f"stage '{sec[6:]}' is missing its kind")
        try:
            sk = StageKind(kind)
        except ValueError:
            raise E.BadParams(f"unknown stage kind '{kind}'") from None
        stages.append(StageSpec(sec[6:], sk, opts))
    return PipelineSpec(pid, tuple(stages))


# ------------------------------------------------------------------ compress

def _check_stage_params(spec: PipelineSpec):
    """Validate string params the way the reference stage bodies would."""
    for st in spec.stages:
        if st.kind == StageKind.PREPROCESS and st.param("op", "identity") != "identity":
            raise E.StageError(st.name, ValueError(f"unsupported preprocess op '{st.param('op')}'"))
    pst = spec.stage_of(StageKind.PREDICT)
    if spec.predictor not in ("lorenzo", "interp", "dualquant"):
        raise E.StageError(pst.name, ValueError(f"unknown predictor '{spec.predictor}'"))
    an = spec.stage_of(StageKind.ANALYSIS)
    if an is not None:
        method = an.param("method", "exact")
        if method not in ("exact", "topk"):
            raise E.StageError(an.name, ValueError(f"unknown histogram method '{method}'"))
        if method == "topk":
            k = int(an.param("k", "16"))
            if not 1 <= k <= 2 * spec.radius():
                raise E.StageError(an.name, ValueError(f"k must be in [1, {2 * spec.radius()}], got {k}"))
    pc = spec.stage_of(StageKind.PRIMARY_CODEC)
    if spec.primary_codec not in ("huffman", "bitshuffle"):
        raise E.StageError(pc.name, ValueError(f"unknown primary codec '{spec.primary_codec}'"))
    if spec.primary_codec == "bitshuffle" and spec.radius() > 32768:
        raise E.StageError(pc.name, E.RadiusTooLarge(f"radius {spec.radius()} exceeds 16-bit code width"))


def _to_device(field) -> torch.Tensor:
    """H2D of the field; direct async copy when the numpy data lives in pinned memory."""
    eng = default_engine()
    src = torch.from_numpy(field.data)
    if src.is_pinned():
        buf = eng.buf("field_in", 4 * field.len)
        dst = buf[: 4 * field.len].view(torch.float32)
        with torch.cuda.stream(eng.stream):
            dst.copy_(src, non_blocking=True)
        return dst
    buf = eng.upload("field_in", field.data)
    return buf[: 4 * field.len].view(torch.float32)


def compress_device(x: torch.Tensor, dims, eb: ErrorBoundSpec, pipeline, *, graph: bool = False,
                    timings: dict | None = None) -> Archive:
    """Compress a device-resident f32 tensor (the timed path).  graph=True
    replays the whole device DAG as one captured CUDA graph (graph_engine();
    `x` is then the graph's static input: keep passing the same tensor).
    `timings` receives per-stage seconds keyed by stage name, as the
    reference's compress_with_timing (pipeline.py:345-379)."""

    spec = get_pipeline(pipeline)
    _check_stage_params(spec)
    eng = graph_engine() if graph else default_engine()
    pred = spec.predictor
    cfg = spec.interp_config() if pred == "interp" else None
    if pred == "interp" and not interp_applicable(dims, cfg.anchor_stride):
        log.warning("interpolation needs a 2D or 3D field with every extent >= %d, got dims %s; "
                    "falling back to Lorenzo", cfg.anchor_stride + 1, tuple(dims))
    prof = pred == "interp" and spec.stage_of(StageKind.PREDICT).param("profile", "0") == "1"
    if prof and graph:   # the profiled choice is a host decision mid-DAG: run eagerly
        eng, graph = default_engine(), False
    run = eng.compress_graphed if graph else eng.compress
    if timings is not None and not graph:
        eng.marks = {}
    try:
        kwx = dict(profile=True) if prof else {}
        da = run(x, dims, int(eb.mode), float(eb.magnitude), pipeline_id=spec.id, predictor=pred,
                 codec=spec.primary_codec, radius=spec.radius(), anchor_stride=cfg.anchor_stride if cfg else 16, **kwx)
        return _archive_of(eng, da, spec, eb, dims, timings)
    finally:
        eng.marks = None


def _span(marks: dict, a: str, b: str) -> float:
    return marks[a].elapsed_time(marks[b]) / 1e3 if a in marks and b in marks else 0.0


def _device_error_stage(spec: PipelineSpec, status: int) -> str:
    """The stage a compress-side device status bit belongs to: a code outside
    the alphabet is the histogram's CodeOutOfRange (encode.py:79-84) when an
    analysis stage runs, everything else the primary codec's."""
    from . import _lib
    an = spec.stage_of(StageKind.ANALYSIS)
    if an is not None and status & _lib.ERR_CODE_RANGE:
        return an.name
    return spec.stage_of(StageKind.PRIMARY_CODEC).name


def _archive_of(eng, da, spec: PipelineSpec, eb: ErrorBoundSpec, dims, timings: dict | None = None) -> Archive:
    """finish() one device result into an Archive (pipeline.py:300-342)."""
    try:
        lo, hi, segs, wire = eng.finish(da)
    except E.FZError as e:
        st = eng.sizes(da)["status"]
        raise E.StageError(_device_error_stage(spec, st), e) from e
    if lo == hi:
        return Archive(spec.id, eb.mode, eb.magnitude, lo, hi, tuple(dims), spec.radius(), ())
    ResolvedBound(eb_from_range(eb.mode, eb.magnitude, lo, hi), lo, hi)
    if timings is not None and eng.marks is not None:
        m = eng.marks
        for st in spec.stages:
            if st.kind == StageKind.PREPROCESS:
                timings[st.name] = 0.0   # identity (pipeline.py:260-264)
        timings[spec.stage_of(StageKind.PREDICT).name] = _span(m, "predict", "predict_end")
        an = spec.stage_of(StageKind.ANALYSIS)
        if an is not None:
            timings[an.name] = _span(m, "predict_end", "primary")
        # primary codec: build + encode, and the D2H that makes its segments host bytes
        timings[spec.stage_of(StageKind.PRIMARY_CODEC).name] = \
            _span(m, "primary", "primary_end") + _span(m, "d2h", "d2h_end")
    sc = spec.stage_of(StageKind.SECONDARY_CODEC)
    if sc is not None:
        t0 = time.perf_counter()
        nprim = 2
        head, prim = segs[:-nprim], segs[-nprim:]
        try:
            cid = int(sc.param("codec_id", "0"))
            prim = [(SEG_SECONDARY_WRAPPED, bytes([k]) + secondary.secondary_encode(p, cid)) for k, p in prim]
        except Exception as e:
            raise E.StageError(sc.name, e) from e
        segs = head + prim
        wire = None
        if timings is not None:
            timings[sc.name] = time.perf_counter() - t0
    a = Archive(spec.id, eb.mode, eb.magnitude, lo, hi, tuple(dims), spec.radius(), tuple(segs))
    if wire is not None:
        attach_wire(a, wire[0].numpy(), wire[1])
    return a


def compress_with_timing(field: Field, eb: ErrorBoundSpec, pipeline):
    """pipeline.py:345-379: the archive plus per-stage seconds keyed by the
    spec's stage names (CUDA-event spans of each stage's kernels; the
    primary codec includes the D2H of its segments).  A constant field
    returns an empty dict, as the reference does."""
    timings: dict = {}
    x = _to_device(field)
    a = compress_device(x, field.dims, eb, pipeline, timings=timings)
    return a, timings


def compress(field: Field, eb: ErrorBoundSpec, pipeline) -> Archive:
    return compress_device(_to_device(field), field.dims, eb, pipeline)


def compress_via_graph(field: Field, eb: ErrorBoundSpec, pipeline, workers: int | None = None) -> Archive:
    """Graph variant (pipeline.py:650-660): the device DAG (predict ->
    serialize-outliers || analysis -> primary-encode) runs as one CUDA graph,
    captured per shape / bound / pipeline on first use and replayed for
    later fields (the H2D lands in the graph's static input).  Archives are
    byte-identical to compress(); `workers` has no GPU meaning."""
    eng = graph_engine()
    x = eng.buf("graph_in_%s" % "x".join(map(str, field.dims)), 4 * field.len)[: 4 * field.len].view(torch.float32)
    src = torch.from_numpy(field.data)
    with torch.cuda.stream(eng.stream):
        x.copy_(src, non_blocking=src.is_pinned())
    return compress_device(x, field.dims, eb, pipeline, graph=True)


# ---------------------------------------------------------------- decompress

def _unwrap(a: Archive) -> dict:
    segs = {}
    for kind, payload in a.segments:
        if kind == SEG_SECONDARY_WRAPPED:
            if len(payload) < 2:
                raise E.CorruptPayload("wrapped segment too short")
            segs[payload[0]] = secondary.secondary_decode(payload[1:])
        else:
            segs[kind] = payload
    return segs


def _outliers(segs: dict, n: int):
    if SEG_OUTLIER_INDICES not in segs or SEG_OUTLIER_VALUES not in segs:
        raise E.CorruptPayload("outlier segments missing")
    ib, vb = segs[SEG_OUTLIER_INDICES], segs[SEG_OUTLIER_VALUES]
    if len(ib) % 8 or len(vb) % 4 or len(ib) // 8 != len(vb) // 4:
        raise E.CorruptPayload("outlier index/value segments disagree")
    idx = np.frombuffer(ib, "<u8")
    vals = np.frombuffer(vb, "<f4")
    if idx.size and int(idx.max()) >= n:
        raise E.CorruptPayload("outlier index out of range")
    return idx, vals


def _codec_segments(spec: PipelineSpec, segs: dict, radius: int):
    """Host-side structural checks of _decode_codes (pipeline.py:415-430)."""
    codec = spec.primary_codec
    if codec == "huffman":
        if SEG_HUFFMAN_CODEBOOK not in segs or SEG_HUFFMAN_BITSTREAM not in segs:
            raise E.CorruptPayload("Huffman segments missing")
        from .encode import HuffmanCodebook
        cb = HuffmanCodebook.from_bytes(segs[SEG_HUFFMAN_CODEBOOK])
        if cb.code_lengths.size != 2 * radius:
            raise E.CorruptPayload(f"codebook covers {cb.code_lengths.size} symbols, alphabet is {2 * radius}")
        if radius > 32768:
            raise E.RadiusTooLarge(f"radius {radius} exceeds the device path's 16-bit codes")
        return {"codebook": cb.code_lengths, "stream": segs[SEG_HUFFMAN_BITSTREAM]}
    if codec == "bitshuffle":
        if SEG_BITSHUFFLE_BITMAP not in segs or SEG_BITSHUFFLE_PAYLOAD not in segs:
            raise E.CorruptPayload("bitshuffle segments missing")
        if radius > 32768:
            raise E.RadiusTooLarge(f"radius {radius} exceeds 16-bit code width")
        return {"bitmap": segs[SEG_BITSHUFFLE_BITMAP], "payload": segs[SEG_BITSHUFFLE_PAYLOAD]}
    raise ValueError(f"unknown primary codec '{codec}'")


def _raise_decode_status(status: int):
    from . import _lib
    if not status:
        return
    try:
        _lib.raise_codec_status(status)
    except E.FZError as e:
        raise E.StageError("decode-codes", e) from e
    if status & (_lib.ERR_OUTLIER_CODE | _lib.ERR_OUTLIER_ORDER):
        raise E.MalformedCodes("outlier position without sentinel code")
    if status & _lib.ERR_HF_SYNC:
        raise RuntimeError("Huffman decoder did not synchronise (increase iterations)")
    raise RuntimeError(f"device status {status:#x}")


def _decompress_dev(a: Archive, pipeline=None, *, graph: bool = False, timings: dict | None = None):
    """Shared body of decompress_device / decompress_with_timing /
    decompress_via_graph: host checks, then the two-stream device DAG.
    Returns (engine, device recon) or (None, constant value)."""
    spec = get_pipeline(pipeline if pipeline is not None else a.pipeline_id)
    n = a.element_count
    if len(a.segments) == 0:
        if a.data_min != a.data_max:
            raise E.CorruptPayload("no segments but the header spans a value range")
        return None, a.data_min
    bound = a.resolved_bound()
    t0 = time.perf_counter()
    segs = _unwrap(a)
    if timings is not None:
        timings["unwrap"] = time.perf_counter() - t0
    radius = a.radius
    try:
        csegs = _codec_segments(spec, segs, radius)
    except Exception as e:
        raise E.StageError("decode-codes", e) from e
    try:
        idx, vals = _outliers(segs, n)
    except Exception as e:
        raise E.StageError("decode-outliers", e) from e
    if idx.size > 1 and not bool(np.all(idx[1:] > idx[:-1])):
        raise E.MalformedCodes("outlier indices not strictly increasing")
    anchors = segs.get(SEG_ANCHOR_GRID, b"")
    pred = spec.predictor
    deltas = None
    if pred == "dualquant":
        db = segs.get(SEG_DQ_DELTAS)
        if db is None or len(db) != 4 * idx.size:
            raise E.StageError("decode-outliers", E.CorruptPayload("dual-quant delta segment missing or sized wrong"))
        deltas = np.frombuffer(db, "<i4")
    stride = spec.interp_config().anchor_stride if pred == "interp" else 16
    weights = None
    pb = segs.get(SEG_INTERP_PROFILE)
    if pred == "interp" and pb is not None:   # opt-in pipeline 5: the profiled choice
        from .device import PROFILE_STRIDES, PROFILE_WEIGHTS
        if len(pb) != 2 or pb[0] not in PROFILE_STRIDES or pb[1] > 2:
            raise E.StageError("reconstruct", E.CorruptPayload("bad interpolation profile segment"))
        stride, weights = pb[0], PROFILE_WEIGHTS[pb[1]]
    if pred == "interp" and len(anchors):
        from .device import pad3
        d3 = pad3(a.dims)
        want = 4 * int(np.prod([(d - 1) // stride + 1 for d in d3]))
        if len(anchors) != want:
            raise E.StageError("reconstruct", E.AnchorSizeMismatch(
                f"anchor payload is {len(anchors)} bytes, expected {want}"))
    eng = graph_engine() if graph else default_engine()
    if timings is not None and not graph:
        eng.marks = {}
    try:
        dag = eng.decompress_dag_graphed if graph else eng.decompress_dag
        try:
            kwd = dict(weights=weights) if weights is not None else {}
            recon = dag(spec.primary_codec, pred, csegs, idx, vals, anchors, a.dims, bound.eb_abs, radius, stride,
                        deltas=deltas, **kwd)
        except E.FZError as e:
            raise E.StageError("decode-codes", e) from e
        return eng, recon
    finally:
        if timings is not None and eng.marks is not None:
            eng._mark("reconstruct_end")
            eng.stream.synchronize()
            m = eng.marks
            timings["decode-codes"] = _span(m, "decode-codes", "decode-codes_end")
            timings["decode-outliers"] = _span(m, "decode-outliers", "decode-outliers_end")
            timings["reconstruct"] = _span(m, "reconstruct", "reconstruct_end")
        eng.marks = None


def decompress_device(a: Archive, pipeline=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """Decompress into a device f32 tensor (the timed path)."""
    eng, recon = _decompress_dev(a, pipeline)
    if eng is None:
        dev = default_engine().device
        t = out if out is not None else torch.empty(a.element_count, dtype=torch.float32, device=dev)
        t.fill_(recon)
        return t
    _raise_decode_status(eng.decode_status())
    if out is not None:
        with torch.cuda.stream(eng.stream):
            out.copy_(recon)
        return out
    with torch.cuda.stream(eng.stream):
        return recon.clone()


def _to_host(a: Archive, eng, recon, t_reconstruct: dict | None = None) -> Field:
    if eng is None:
        return Field(a.dims, np.full(a.element_count, recon, np.float32))
    t0 = time.perf_counter()
    host = torch.empty(recon.numel(), dtype=torch.float32, pin_memory=True)
    with torch.cuda.stream(eng.stream):
        host.copy_(recon, non_blocking=True)
    eng._sync()
    if t_reconstruct is not None and "reconstruct" in t_reconstruct:
        t_reconstruct["reconstruct"] += time.perf_counter() - t0
    _raise_decode_status(eng.decode_status())
    # the decoder output is finite by construction; skip Field's O(n) host re-validation
    return Field.trusted(a.dims, host.numpy())


def decompress_with_timing(a: Archive, pipeline=None):
    """pipeline.py:439-466: the field plus seconds for "unwrap",
    "decode-codes", "decode-outliers" (both branches of the two-stream DAG,
    which overlap) and "reconstruct" (predictor inverse + D2H)."""
    timings: dict = {}
    eng, recon = _decompress_dev(a, pipeline, timings=timings)
    return _to_host(a, eng, recon, timings), timings


def decompress(a: Archive, pipeline=None) -> Field:
    eng, recon = _decompress_dev(a, pipeline)
    return _to_host(a, eng, recon)


# ------------------------------------------------------------------- batches
# Several same-shaped fields at once ("several fields in flight
# per GPU"): one batched Lorenzo wavefront interleaves all members' tiles, so
# the GPU is busier than with one field at a time.  Archives and
# reconstructions are identical to per-field compress()/decompress().

def _batchable(spec: PipelineSpec, dims, n: int) -> bool:
    return spec.predictor == "lorenzo" and len(dims) > 1 and n % 64 == 0


def compress_batch(fields: list, eb: ErrorBoundSpec, pipeline) -> list:
    """compress() of every field; same-shaped Lorenzo fields share one launch."""
    spec = get_pipeline(pipeline)
    _check_stage_params(spec)
    if not fields:
        return []
    dims = tuple(fields[0].dims)
    n = fields[0].len
    if len(fields) == 1 or any(tuple(f.dims) != dims for f in fields) or not _batchable(spec, dims, n):
        return [compress(f, eb, pipeline) for f in fields]
    eng = default_engine()
    X = eng.buf("cb_in", 4 * n * len(fields))[: 4 * n * len(fields)].view(torch.float32).view(len(fields), n)
    for i, f in enumerate(fields):
        src = torch.from_numpy(f.data)
        if not src.is_pinned():
            src = eng.pinned(f"cb_stage#{i}", 4 * n)[: 4 * n].view(torch.float32).copy_(src)
        with torch.cuda.stream(eng.stream):
            X[i].copy_(src, non_blocking=True)
    das = eng.compress_batch(X, dims, int(eb.mode), float(eb.magnitude), pipeline_id=spec.id,
                             predictor=spec.predictor, codec=spec.primary_codec, radius=spec.radius())
    return [_archive_of(eng, da, spec, eb, dims) for da in das]


def decompress_batch(archives: list, pipeline=None) -> list:
    """decompress() of every archive; same-shaped Lorenzo archives share one
    batched wavefront (each member's codec decode and outlier scatter first)."""
    if not archives:
        return []
    a0 = archives[0]
    spec = get_pipeline(pipeline if pipeline is not None else a0.pipeline_id)
    n = a0.element_count
    same = all(a.dims == a0.dims and a.pipeline_id == a0.pipeline_id and a.radius == a0.radius and len(a.segments)
               for a in archives)
    if len(archives) == 1 or not same or not _batchable(spec, a0.dims, n) or \
            any(SEG_ANCHOR_GRID in _unwrap(a) for a in archives):
        return [decompress(a, pipeline) for a in archives]
    eng = default_engine()
    F = len(archives)
    nw = (n + 31) // 32
    codes = eng.buf("db_codes", 2 * F * n + 16)
    bitmap = eng.buf("db_bitmap", 4 * F * nw, zero=True)
    OUT = eng.buf("db_out", 4 * F * n)[: 4 * F * n].view(torch.float32).view(F, n)
    radius = a0.radius
    codec = spec.primary_codec
    ebs = []
    for f, a in enumerate(archives):
        tag = f"#{f}"
        segs = _unwrap(a)
        try:
            if radius > 32768:
                raise E.RadiusTooLarge(f"radius {radius} exceeds the device path's 16-bit codes")
            if codec == "huffman":
                if SEG_HUFFMAN_CODEBOOK not in segs or SEG_HUFFMAN_BITSTREAM not in segs:
                    raise E.CorruptPayload("Huffman segments missing")
                from .encode import HuffmanCodebook
                cb = HuffmanCodebook.from_bytes(segs[SEG_HUFFMAN_CODEBOOK])
                if cb.code_lengths.size != 2 * radius:
                    raise E.CorruptPayload(f"codebook covers {cb.code_lengths.size} symbols, alphabet is {2 * radius}")
                eng.decode_codes("huffman", {"codebook": cb.code_lengths, "stream": segs[SEG_HUFFMAN_BITSTREAM]}, n,
                                 radius, tag=tag, codes_out=codes[2 * n * f:2 * n * (f + 1)])
            else:
                if SEG_BITSHUFFLE_BITMAP not in segs or SEG_BITSHUFFLE_PAYLOAD not in segs:
                    raise E.CorruptPayload("bitshuffle segments missing")
                eng.decode_codes("bitshuffle", {"bitmap": segs[SEG_BITSHUFFLE_BITMAP],
                                                "payload": segs[SEG_BITSHUFFLE_PAYLOAD]}, n, radius, tag=tag,
                                 codes_out=codes[2 * n * f:2 * n * (f + 1)])
        except Exception as e:
            raise E.StageError("decode-codes", e) from e
        try:
            idx, vals = _outliers(segs, n)
        except Exception as e:
            raise E.StageError("decode-outliers", e) from e
        if idx.size > 1 and not bool(np.all(idx[1:] > idx[:-1])):
            raise E.MalformedCodes("outlier indices not strictly increasing")
        eb_abs = a.resolved_bound().eb_abs
        ebs.append(eb_abs)
        eng.reconstruct("lorenzo", codes[2 * n * f:2 * n * (f + 1)], idx, vals, b"", a.dims, eb_abs, radius,
                        out=OUT[f], tag=tag, bitmap_out=bitmap[4 * nw * f:4 * nw * (f + 1)])
    from .device import pad3
    n0, n1, n2 = pad3(a0.dims)
    ebt = eng.upload("db_eb", np.asarray(ebs, np.float64))
    ws = eng.buf("db_lzws", eng.lib.fzb_lorenzo_batch_workspace_bytes(F, n0, n1, n2), zero_new=True)
    from .device import _p
    eng._call("fzb_lorenzo_decode_batch_f32", _p(codes), _p(bitmap), nw, _p(OUT), F, n, n0, n1, n2, _p(ebt), radius,
              _p(ws), ws.numel(), eng.sp, nk=2)
    from . import _lib
    out = []
    for f, a in enumerate(archives):
        status = eng.decode_status(f"#{f}")
        if status:
            try:
                _lib.raise_codec_status(status)
            except E.FZError as e:
                raise E.StageError("decode-codes", e) from e
            if status & (_lib.ERR_OUTLIER_CODE | _lib.ERR_OUTLIER_ORDER):
                raise E.MalformedCodes("outlier position without sentinel code")
            raise RuntimeError(f"device status {status:#x}")
        host = torch.empty(n, dtype=torch.float32, pin_memory=True)
        with torch.cuda.stream(eng.stream):
            host.copy_(OUT[f], non_blocking=True)
        out.append((a.dims, host))
    eng._sync()
    return [Field.trusted(d, h.numpy()) for d, h in out]


def worker_count(requested: int | None = None) -> int:
    """pipeline.py:477-487 (FZPIPE_THREADS caps the worker count)."""
    base = requested if requested is not None else (os.cpu_count() or 1)
    cap = os.environ.get("FZPIPE_THREADS")
    if cap is not None:
        try:
            base = min(base, max(1, int(cap)))
        except ValueError:
            pass
    return max(1, base)


def decompress_via_graph(a: Archive, workers: int | None = None) -> Field:
    """Graph variant (pipeline.py:583-591): the four-task decompress graph
    (parse -> huffman-decode || outlier-scatter -> predict-reconstruct) as a
    captured two-stream CUDA graph, replayed for later archives of the same
    shape and payload sizes; bitwise equal to decompress().  As in the
    reference, it applies to every pipeline here (a bitshuffle decode is the
    same fork with another codec branch); `workers` has no GPU meaning."""
    eng, recon = _decompress_dev(a, graph=True)
    return _to_host(a, eng, recon)
