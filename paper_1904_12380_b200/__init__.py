"""B200-native fp32 row softmax -- drop-in for softmax_kit's softmax entry point.

Reference: /root/reference/pkg/src/softmax_kit/kernels.py:350-362
(``softmax(m: Matrix2D, variant: KernelVariant, cfg: LaneConfig) -> Matrix2D``).
The numeric work runs in hand-written sm_100a kernels behind the C ABI in
include/softmax_b200.h (libsoftmax_b200.so); this package is the host-side
mirror of the reference interface.  There is no CPU fallback.
"""

from .errors import ArgumentError, NumericDomainError, ResourceError, SoftmaxKitError
from .lanes import LaneConfig
from .tensor import FillSpec, Matrix2D, alloc_matrix, fill_uniform
from . import components
from .components import (
    exp_batch,
    row_max_scalar,
    row_stats,
    row_sum_scalar,
    scale_reciprocal,
    subtract_broadcast,
    value_clip,
)
from .kernels import (
    CLIP_FLOOR,
    FLT_MIN_NORMAL,
    LADDER,
    KernelVariant,
    RowStats,
    row_stats_device,
    softmax,
    softmax_into,
    variant_mode,
)

__all__ = [
    "ArgumentError",
    "NumericDomainError",
    "ResourceError",
    "SoftmaxKitError",
    "LaneConfig",
    "FillSpec",
    "Matrix2D",
    "alloc_matrix",
    "fill_uniform",
    "CLIP_FLOOR",
    "FLT_MIN_NORMAL",
    "LADDER",
    "KernelVariant",
    "RowStats",
    "row_stats_device",
    "softmax",
    "softmax_into",
    "variant_mode",
    "components",
    "row_max_scalar",
    "subtract_broadcast",
    "value_clip",
    "exp_batch",
    "row_sum_scalar",
    "scale_reciprocal",
    "row_stats",
]
