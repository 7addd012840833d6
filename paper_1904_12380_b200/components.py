"""The reference's 1-D component operations, computed on the GPU.

Reference: /root/reference/pkg/src/softmax_kit/kernels.py:220-276 -- the
spec-level building blocks softmax is made of (row max, shift, ValueClip,
exp, wide row sum, reciprocal scale, and the (max, exp-sum) RowStats pair).
Same names, argument checks and error classes; the arithmetic runs in this
library's kernels (include/softmax_b200.h):

    row_max_scalar    sk_row_stats_f32 (max part)   exact: max is order-free
    subtract_broadcast sk_shift_scale_f32 (scale 1) exact IEEE x - v
    exp_batch         sk_exp_f32                   <= 2.53 ulp (np.exp: <= ~3)
    row_sum_scalar    sk_row_sum_f32               f64 accumulation, rounded to f32
    scale_reciprocal  sk_shift_scale_f32 (shift 0) exact IEEE x * (1/(float)s)
    row_stats         sk_row_stats_f32             (max, sum exp(x - max)), unclipped

A numpy row is copied to the current CUDA device and the result copied back
(numpy in, numpy out, like the reference); a CUDA tensor stays on its device
and results come back as CUDA tensors.  There is no CPU fallback: without a
GPU every call raises SoftmaxKitError.  ``value_clip`` is the scalar clamp
rule itself (no array work), kept for API parity.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .errors import ArgumentError, NumericDomainError
from .kernels import CLIP_FLOOR, RowStats, _bad_flag, _require_cuda, _torch

__all__ = [
    "row_max_scalar",
    "subtract_broadcast",
    "value_clip",
    "exp_batch",
    "row_sum_scalar",
    "scale_reciprocal",
    "row_stats",
]


def _as_row(row, op: str):
    """(device tensor, came_from_host) with the reference's checks
    (kernels.py:220-226): 1-D, non-empty, float32."""
    torch = _torch()
    if isinstance(row, torch.Tensor):
        if not row.is_cuda:
            raise ArgumentError(f"{op}: torch input must be a CUDA tensor (there is no CPU path)")
        if row.dim() != 1:
            raise ArgumentError(f"{op} expects a 1-D row, got ndim={row.dim()}")
        if row.numel() == 0:
            raise ArgumentError(f"{op} requires a non-empty row")
        return row.to(torch.float32).contiguous(), False
    a = np.ascontiguousarray(row, dtype=np.float32)
    if a.ndim != 1:
        raise ArgumentError(f"{op} expects a 1-D row, got ndim={a.ndim}")
    if a.size == 0:
        raise ArgumentError(f"{op} requires a non-empty row")
    _require_cuda()
    return torch.from_numpy(a).to(torch.device("cuda", torch.cuda.current_device())), True


def _stream(t):
    return _torch().cuda.current_stream(t.device).cuda_stream


def _stats(x, op: str):
    """sk_row_stats_f32 on a 1 x C row, unclipped (row_stats kernels.py:272-276)."""
    torch = _torch()
    rmax = torch.empty(1, dtype=torch.float32, device=x.device)
    rsum = torch.empty(1, dtype=torch.float64, device=x.device)
    with torch.cuda.device(x.device):
        flag = _bad_flag(torch, x.device)
        _native.check(_native.lib().sk_row_stats_f32(
            x.data_ptr(), 1, x.numel(), x.numel(), _native.SK_MODE_EXACT, rmax.data_ptr(),
            rsum.data_ptr(), flag.data_ptr(), None, 0, _stream(x)), op)
        if int(flag.item()) != -1:
            # a NaN / inf in the row: the reference returns its scan result
            # (no error), so recompute with the NaN / inf-propagating kernel
            flag.fill_(-1)
            _native.check(_native.lib().sk_row_stats_ref_f32(
                x.data_ptr(), x.numel(), rmax.data_ptr(), rsum.data_ptr(), _stream(x)), op)
    return rmax, rsum


def row_max_scalar(row):
    """Row maximum (kernels.py:229-231; the strict left-to-right scan there --
    the maximum of finite values does not depend on the order)."""
    x, host = _as_row(row, "row_max_scalar")
    rmax, _ = _stats(x, "row_max_scalar")
    return np.float32(rmax.item()) if host else rmax[0]


def subtract_broadcast(row, v: float):
    """``row - v`` elementwise, exact IEEE subtraction (kernels.py:234-236)."""
    torch = _torch()
    x, host = _as_row(row, "subtract_broadcast")
    y = torch.empty_like(x)
    with torch.cuda.device(x.device):
        _native.check(_native.lib().sk_shift_scale_f32(
            x.data_ptr(), y.data_ptr(), x.numel(), float(np.float32(v)), 1.0, _stream(x)),
            "subtract_broadcast")
    return y.cpu().numpy() if host else y


def value_clip(x: float) -> np.float32:
    """Clamp a shifted logit at the -64 floor (kernels.py:239-242): the rule
    every clipped kernel applies (kClipFloor in csrc/sk_common.cuh)."""
    x32 = np.float32(x)
    return x32 if x32 > CLIP_FLOOR else CLIP_FLOOR


def exp_batch(buf):
    """In-place elementwise exponential of a float32 buffer (kernels.py:245-255),
    as one device call (sk_exp_f32)."""
    torch = _torch()
    if isinstance(buf, torch.Tensor):
        if not buf.is_cuda:
            raise ArgumentError("exp_batch: torch input must be a CUDA tensor (there is no CPU path)")
        if buf.dtype != torch.float32:
            raise ArgumentError(f"exp_batch expects float32, got {buf.dtype}")
        if not buf.is_contiguous():
            raise ArgumentError("exp_batch expects a contiguous buffer")
        with torch.cuda.device(buf.device):
            _native.check(_native.lib().sk_exp_f32(buf.data_ptr(), buf.numel(),
                                                   _native.SK_MODE_EXACT, _stream(buf)),
                          "exp_batch")
        return buf
    b = np.asarray(buf)
    if b.dtype != np.float32:
        raise ArgumentError(f"exp_batch expects float32, got {b.dtype}")
    if b.size == 0:
        return b
    _require_cuda()
    d = torch.from_numpy(np.ascontiguousarray(b).reshape(-1)).to(
        torch.device("cuda", torch.cuda.current_device()))
    with torch.cuda.device(d.device):
        _native.check(_native.lib().sk_exp_f32(d.data_ptr(), d.numel(), _native.SK_MODE_EXACT,
                                               _stream(d)), "exp_batch")
    b[...] = d.cpu().numpy().reshape(b.shape)
    return b


def row_sum_scalar(row):
    """Row sum accumulated in double, rounded to float32 (kernels.py:258-260)."""
    torch = _torch()
    x, host = _as_row(row, "row_sum_scalar")
    s = torch.empty(1, dtype=torch.float64, device=x.device)
    with torch.cuda.device(x.device):
        _native.check(_native.lib().sk_row_sum_f32(x.data_ptr(), 1, x.numel(), x.numel(),
                                                   s.data_ptr(), _stream(x)), "row_sum_scalar")
    return np.float32(s.item()) if host else s.to(torch.float32)[0]


def scale_reciprocal(row, sum: float):
    """``row * (1/sum)``: one fp32 reciprocal, then IEEE multiplies
    (kernels.py:263-269); a non-finite or non-positive sum raises
    NumericDomainError."""
    torch = _torch()
    x, host = _as_row(row, "scale_reciprocal")
    s = np.float32(sum)
    if not np.isfinite(s) or s <= 0:
        raise NumericDomainError(f"normalization sum must be finite and > 0, got {sum}")
    r = np.float32(1.0) / s
    y = torch.empty_like(x)
    with torch.cuda.device(x.device):
        _native.check(_native.lib().sk_shift_scale_f32(
            x.data_ptr(), y.data_ptr(), x.numel(), 0.0, float(r), _stream(x)), "scale_reciprocal")
    return y.cpu().numpy() if host else y


def row_stats(row) -> RowStats:
    """(max, sum exp(row - max)) of one row, unclipped like the reference
    (kernels.py:272-276); the sum is accumulated in double and rounded to
    float32.  The 2-D device form is kernels.row_stats_device."""
    x, host = _as_row(row, "row_stats")
    rmax, rsum = _stats(x, "row_stats")
    if host:
        return RowStats(max=np.float32(rmax.item()), sum=np.float32(rsum.item()))
    return RowStats(max=rmax[0], sum=rsum.to(rmax.dtype)[0])
