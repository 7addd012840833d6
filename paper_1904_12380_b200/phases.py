"""GPU phase pipeline: the reference's plugin point, phase by phase.

Mirror of ``PhasePipeline`` / ``variant_pipeline`` (reference
kernels.py:283-339): the three phases of one softmax bound to a shape, here
as three separate sm_100a kernels over CUDA tensors (sk_maxsub_f32,
sk_exp_f32, sk_sumscale_f32).  The fused ``softmax()`` is the hot path; this
unfused pipeline exists for the phase profile (profiler.time_phases, Fig. 2)
and for callers that drive the phases themselves, as the reference's timers
do (profiler.py:112-130, 148-160).

``maxsub(src, dst)`` reads logits and writes shifted (clipped) logits;
``exp(buf)`` and ``sumscale(buf)`` transform ``dst`` in place.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

from . import _native
from .errors import ArgumentError
from .kernels import KernelVariant, LaneConfig, variant_mode


@dataclass(frozen=True)
class PhasePipeline:
    variant: KernelVariant
    maxsub: Callable
    exp: Callable
    sumscale: Callable


def _stream(t):
    import torch

    return torch.cuda.current_stream(t.device).cuda_stream


def _check(t, rows, cols, what):
    import torch

    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32:
        raise ArgumentError(f"{what} must be a float32 CUDA tensor")
    if t.numel() != rows * cols or not t.is_contiguous():
        raise ArgumentError(f"{what} must be contiguous with {rows}x{cols} elements")


def variant_pipeline(variant: KernelVariant, rows: int, cols: int,
                     cfg: LaneConfig = LaneConfig()) -> PhasePipeline:
    """Bind a variant's three phase kernels to a shape (kernels.py:297-339)."""
    mode = variant_mode(variant)
    if not isinstance(cfg, LaneConfig):
        raise ArgumentError(f"expected a LaneConfig, got {cfg!r}")
    if rows < 1 or cols < 1:
        raise ArgumentError(f"matrix dimensions must be >= 1, got {rows}x{cols}")
    from . import kernels

    L = _native.lib()

    def maxsub(src, dst):
        _check(src, rows, cols, "src")
        _check(dst, rows, cols, "dst")
        clip = 1 if variant is KernelVariant.REFERENCE_CLIPPED else 0
        if kernels._SKIP_MAX_SHIFT:  # kernels.py:309-311: the shift becomes a plain copy
            dst.copy_(src.view_as(dst))
            return
        _native.check(L.sk_maxsub_f32(src.data_ptr(), dst.data_ptr(), rows, cols, cols, cols,
                                      clip, _stream(src)), "maxsub")

    def exp(buf):
        _check(buf, rows, cols, "buf")
        _native.check(L.sk_exp_f32(buf.data_ptr(), rows * cols, mode, _stream(buf)), "exp")

    def sumscale(buf):
        _check(buf, rows, cols, "buf")
        _native.check(L.sk_sumscale_f32(buf.data_ptr(), rows, cols, cols, _stream(buf)),
                      "sumscale")

    return PhasePipeline(variant=variant, maxsub=maxsub, exp=exp, sumscale=sumscale)
