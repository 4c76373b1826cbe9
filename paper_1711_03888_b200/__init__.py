"""nbz-b200: the nbz SZ-LV / SZ-LV-PRX compression path on B200 (sm_100a).

Drop-in for the reference package's hot path (pkg/src/nbz/pipeline.py):
the same ``compress`` / ``decompress`` / ``ratio`` entry points, options and
exceptions, computed by hand-written CUDA kernels behind a C ABI
(include/nbzg.h, libnbzg.so).  See DESIGN.md.
"""

from .errors import (ArchiveError, BoundTooSmallError, DecodeError, DegenerateRangeError,
                     EncodeError, NbzError, ValidationError)
from .model import (FIELD_NAMES, BoundKind, ErrorBoundSpec, ParticleSnapshot, field_range,
                    resolve_bound)
from .pipeline import (DEFAULT_SETTINGS, GPU_MODES, MODE_ALIASES, Archive, CompressResult, Mode,
                       Settings, Stream, StreamKind, compress, decompress, ratio)
from .rindex import RIndexVariant, Segment

__version__ = "0.1.0"

__all__ = [
    "Archive", "ArchiveError", "BoundKind", "BoundTooSmallError", "CompressResult",
    "DEFAULT_SETTINGS", "DecodeError", "DegenerateRangeError", "EncodeError", "ErrorBoundSpec",
    "FIELD_NAMES", "GPU_MODES", "MODE_ALIASES", "Mode", "NbzError", "ParticleSnapshot",
    "RIndexVariant", "Segment", "Settings", "Stream", "StreamKind", "ValidationError",
    "compress", "decompress", "field_range", "ratio", "resolve_bound", "__version__",
]
