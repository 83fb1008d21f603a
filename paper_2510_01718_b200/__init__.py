"""B200-native basis-decomposed (BD) K/V projection — drop-in for bdattn's hot path.

Mirrors the reference package's names (ref: pkg/src/bdattn/__init__.py:18-91) for
the path BASELINE.json's north star names: ``fused_kv_proj`` (the operator) and its
callers — ``bda_forward`` / ``attention_scores`` (GPU), ``bd_linear_forward`` (GPU) —
the offline preparation ``bda_prepare`` / ``bd_decompose*`` / ``bd_linear_from_lowrank``
(CPU, NumPy/SciPy, the reference's exact operation sequence), the weight carriers, the
error types and the parity harness.  The arithmetic runs in hand-written sm_100a CUDA
kernels behind a C ABI (include/bd_kv_proj.h, libbd_kvproj.so); there is no CPU
fallback on the GPU path.
"""

from .attention import (
    BDAWeights,
    MHAWeights,
    attention_scores,
    bda_forward,
    bda_prepare,
    merge_heads,
    mha_forward,
    select_tag,
)
from .decompose import (
    RANK_DEFICIENCY_TOL,
    Axis,
    BDFactors,
    CostReport,
    LstsqResult,
    Side,
    Tag,
    bd_decompose,
    bd_decompose_both,
    bd_reconstruct,
    cost_report,
    frobenius_norm,
    lstsq,
    ordered_matmul,
)
from .errors import NativeLibraryError, PrecisionError, ShapeError
from .kv_proj import (
    flop_ratio,
    fold_rmsnorm,
    fused_kv_proj,
    fused_kv_proj_grouped,
    fused_rmsnorm_kv_proj_grouped,
    fused_kv_proj_grouped_host,
    fused_kv_proj_host,
    kv_flops,
    tag_offsets,
)
from .linear import (
    BDLinearLayer,
    LowRankLayer,
    bd_linear_forward,
    bd_linear_from_lowrank,
    lowrank_forward,
    matmul,
)
from .tensorio import (
    ManifestError,
    TensorFileError,
    load_bda_manifest,
    load_mha_manifest,
    load_tensor,
    manifest_kind,
    save_bda_manifest,
    save_mha_manifest,
    save_tensor,
)
from .verify import (
    EQUIVALENCE_THRESHOLDS,
    KERNEL_MAXREL,
    ErrorReport,
    Rng,
    Target,
    TrialSummary,
    equivalence_check,
    gen_random_mha,
    max_relative_error,
    rand_gaussian,
    reconstruction_error_report,
)

__version__ = "0.2.0"
