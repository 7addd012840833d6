"""torch.ops.softmax_b200.* -- TORCH_LIBRARY launchers over the C ABI.

SURVEY.md §8(b).2's op surface (sk_torch_ops.cpp): ``softmax_fwd(x, clip)``,
``softmax_fwd_out(x, y, clip)``, ``row_max(x)``, ``row_sumexp(x, gmax, clip)``,
``normalize_(x, gmax, gsum, y, clip)``.  They run on the current CUDA stream,
are capturable in CUDA graphs, and have CUDA kernels only (a CPU tensor
raises: there is no CPU fallback).
"""

from __future__ import annotations

import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parents[1] / "libsoftmax_b200_torch.so"
_lock = threading.Lock()
_loaded = False


def load():
    """Register the ops (idempotent) and return ``torch.ops.softmax_b200``."""
    global _loaded
    import torch

    with _lock:
        if not _loaded:
            if not LIB_PATH.exists():
                raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build()")
            from .. import _native

            _native.lib()  # the C library first, so both share one copy
            torch.ops.load_library(str(LIB_PATH))
            _loaded = True
    return torch.ops.softmax_b200
