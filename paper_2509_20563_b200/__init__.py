"""B200-native (sm_100a) FZModules hot path -- drop-in for the fzpipe API.

Predictor-quantizers (exact Lorenzo 1-3D, G-Interp), histogram, canonical
package-merge Huffman and FZ-GPU bitshuffle run as hand-written CUDA
kernels in libfzb200.so (C ABI: include/fzb200.h); this package mirrors
fzpipe's module/pipeline API on top and produces byte-identical archives.
There is no CPU fallback on any path.
"""

from .core import (  # noqa: F401
    Archive, ErrorBoundSpec, archive_buffer, ErrorMode, Field, QuantOutput, ResolvedBound, field_from_array, parse_archive,
    resolve_bound, serialize_archive,
)
from .errors import FZError  # noqa: F401
from .metrics import QualityReport, RateReport, quality, rate  # noqa: F401
from .pipeline import (  # noqa: F401
    PipelineSpec, StageKind, StageSpec, compress, compress_batch, compress_device, compress_via_graph,
    compress_with_timing, decompress, decompress_batch, decompress_device, decompress_via_graph,
    decompress_with_timing, get_pipeline, load_pipeline_file, register_pipeline, registered_pipelines,
)

__version__ = "0.1.0"
