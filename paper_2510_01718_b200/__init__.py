"""B200-native basis-decomposed (BD) K/V projection — drop-in for bdattn's hot path.

Mirrors the reference package's names (ref: pkg/src/bdattn/__init__.py:18-91) for
the path BASELINE.json's north star names: ``fused_kv_proj`` (the operator),
``Tag``, ``ShapeError``/``PrecisionError``, the BDA weight types, ``bda_prepare``
(offline, CPU) and ``bda_forward`` (GPU).  The projection runs in hand-written
sm_100a CUDA kernels behind a C ABI (include/bd_kv_proj.h).
"""

from .errors import NativeLibraryError, PrecisionError, ShapeError
from .kv_proj import (
    Tag,
    flop_ratio,
    fused_kv_proj,
    fused_kv_proj_grouped,
    fused_kv_proj_grouped_host,
    fused_kv_proj_host,
    kv_flops,
    tag_offsets,
)

__version__ = "0.1.0"
