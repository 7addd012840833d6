"""``LaneConfig`` -- part of the reference entry point's signature.

Reference: /root/reference/pkg/src/softmax_kit/simd_reduce.py:60-75.  The lane
width models x86 register lanes; a GPU warp reduces with its own structure, so
here the value is validated (same rule, same error) but has no numeric effect,
exactly as for the ReferenceClipped rung in the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import ArgumentError


@dataclass(frozen=True)
class LaneConfig:
    """Number of single-precision lanes in the wide path (simd_reduce.py:60-75)."""

    width: int = 8

    def __post_init__(self) -> None:
        if self.width < 4 or self.width & (self.width - 1):
            raise ArgumentError(f"lane width must be a power of two >= 4, got {self.width}")

    @property
    def half_width(self) -> int:
        return self.width // 2
