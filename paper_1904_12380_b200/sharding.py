"""Multi-GPU sharding of the row softmax (one process per GPU, torchrun).

Row sharding (configs c4, c5a): rows are independent, so each rank runs the
single-GPU softmax on its contiguous row block -- no communication in the
data path.  The kernel plan depends only on C (and alignment, which a
contiguous row block preserves when C % 4 == 0), so a row computed on any
rank is bit-identical to the same row computed on one GPU.

Column sharding (config c5b): each rank holds the column block
[N, C_r] of every row.  Only per-row statistics cross NVLink:

    (m_r, s_r)  = local max and local sum of exp(clip(x - m_r))     (K4 stats)
    M           = all_reduce(m_r, MAX)                              (NCCL, N fp32)
    s_r        *= exp(m_r - M)                                      (rescale)
    S           = all_reduce(s_r, SUM)                              (NCCL, N fp64)
    y           = exp(clip(x - M)) * (1 / (float)S)                 (normalize)

This is the RowStats pair of the reference (kernels.py:108-112, 272-276)
merged the way context-parallel attention merges (m, l) partials.  The
collective sequence is expressed against a small ``ColumnShardOps`` interface
so the host logic can be exercised on CPU with gloo and a numpy test double
(tests/test_sharding_gloo.py); the product binds it to the CUDA kernels.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Any, Callable

from .errors import ArgumentError
from .kernels import KernelVariant, LaneConfig, softmax, variant_mode


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block of ``n`` items owned by ``rank``: (start, count).
    The first ``n % world`` ranks get one extra item."""
    if world < 1 or not 0 <= rank < world:
        raise ArgumentError(f"bad rank {rank} for world size {world}")
    if n < 0:
        raise ArgumentError("n must be >= 0")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def row_sharded_softmax(x_local, variant: KernelVariant, cfg: LaneConfig = LaneConfig(), **kw):
    """Softmax of this rank's row block: no collective (rows are independent)."""
    return softmax(x_local, variant, cfg, **kw)


@dataclass
class ColumnShardOps:
    """The three local kernels of the column-sharded softmax."""

    local_stats: Callable[[Any, int], tuple[Any, Any]]      # x -> (m f32[N], s f64[N])
    rescale: Callable[[Any, Any, Any], Any]                 # (m_local, M, s) -> s (in place ok)
    normalize: Callable[[Any, Any, Any, int], Any]          # (x, M, S, mode) -> y


def cuda_column_ops() -> ColumnShardOps:
    """Bind ColumnShardOps to the native kernels (sk_row_stats_f32,
    sk_rescale_sumexp, sk_normalize_f32)."""
    import torch

    from . import _native

    def stream_of(t):
        return torch.cuda.current_stream(t.device).cuda_stream

    def local_stats(x, mode):
        rows, cols = x.shape
        m = torch.empty(rows, dtype=torch.float32, device=x.device)
        s = torch.empty(rows, dtype=torch.float64, device=x.device)
        if rows:
            _native.check(_native.lib().sk_row_stats_f32(
                x.data_ptr(), rows, cols, x.stride(0) if rows > 1 else cols, mode, m.data_ptr(),
                s.data_ptr(), None, None, 0, stream_of(x)), "row_stats")
        return m, s

    def rescale(m_local, M, s):
        _native.check(_native.lib().sk_rescale_sumexp(
            m_local.data_ptr(), M.data_ptr(), s.data_ptr(), s.numel(), stream_of(s)), "rescale")
        return s

    def normalize(x, M, S, mode):
        rows, cols = x.shape
        y = torch.empty_like(x)
        if rows:
            ld = x.stride(0) if rows > 1 else cols
            _native.check(_native.lib().sk_normalize_f32(
                x.data_ptr(), y.data_ptr(), rows, cols, ld, cols, mode, M.data_ptr(),
                S.data_ptr(), stream_of(x)), "normalize")
        return y

    return ColumnShardOps(local_stats, rescale, normalize)


def column_sharded_softmax(x_local, variant: KernelVariant, group=None,
                           ops: ColumnShardOps | None = None, all_reduce=None):
    """Softmax over rows whose columns are split across the ranks of ``group``.

    ``x_local`` is this rank's [N, C_r] block; returns its [N, C_r] output.
    Two latency-bound all-reduces (N fp32 MAX, N fp64 SUM) are the only
    communication.  ``all_reduce(tensor, op_name)`` defaults to
    torch.distributed.all_reduce over ``group``.
    """
    mode = variant_mode(variant)
    if ops is None:
        ops = cuda_column_ops()
    if all_reduce is None:
        import torch.distributed as dist

        def all_reduce(t, op):
            dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM,
                            group=group)
            return t

    m_local, s = ops.local_stats(x_local, mode)
    M = all_reduce(_clone(m_local), "max")
    s = ops.rescale(m_local, M, s)
    S = all_reduce(s, "sum")
    return ops.normalize(x_local, M, S, mode)


def _clone(t):
    return t.clone() if hasattr(t, "clone") else t.copy()
