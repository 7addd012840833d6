"""The drop-in softmax entry point, backed by sm_100a kernels.

Mirror of /root/reference/pkg/src/softmax_kit/kernels.py:

* ``KernelVariant`` / ``LADDER`` (kernels.py:76-96): same members, values and
  ``from_name`` error.
* ``CLIP_FLOOR`` / ``FLT_MIN_NORMAL`` (kernels.py:99-101): same constants; the
  CUDA kernels hard-code the same values (csrc/sk_common.cuh).
* ``softmax(m, variant, cfg=LaneConfig())`` (kernels.py:350-362): same
  signature and error behaviour.  ``m`` may be

  - a ``Matrix2D`` -- this package's, or the reference's own
    ``softmax_kit.tensor.Matrix2D`` (duck-typed: rows / cols / flat float32
    ``data`` / ``view2d``, validated like tensor.py:43-57): copied to the GPU
    in row chunks, computed, copied back into a fresh Matrix2D of the
    caller's class (H2D/compute/D2H pipelined over streams inside the native
    library; pageable buffers are staged through page-locked slots);
  - a CUDA ``torch.Tensor[N, C]`` float32 with unit column stride (the hot
    path): returns a same-shape CUDA tensor on the current stream;
  - a 2-D float32 ``numpy.ndarray``: like ``Matrix2D``, returns an ndarray.

  ``variant`` (this package's KernelVariant or the reference's, matched by
  value) selects the arithmetic: ReferenceClipped clamps shifted logits
  at -64 (kernels.py:147); every other rung is the same math without the clip
  (SPEC.md:97 invariant); FullVectorizedApproxExp uses the ex2.approx
  exponential (tolerance 1e-5, bench.py:52).  ``cfg`` is validated but has no
  numeric effect (as for the scalar rungs in the reference).

There is no CPU fallback: without a CUDA device every call raises
``SoftmaxKitError``.
"""

from __future__ import annotations

import contextlib
import ctypes
import enum
import threading
from typing import Any, NamedTuple

import numpy as np

from . import _native, hostpin
from .errors import ArgumentError, NumericDomainError, SoftmaxKitError
from .lanes import LaneConfig
from .tensor import Matrix2D, alloc_matrix

__all__ = [
    "KernelVariant",
    "LADDER",
    "RowStats",
    "CLIP_FLOOR",
    "FLT_MIN_NORMAL",
    "softmax",
    "softmax_into",
    "variant_mode",
    "LaneConfig",
]


class KernelVariant(enum.Enum):
    """One rung of the optimization ladder (kernels.py:76-93)."""

    REFERENCE_CLIPPED = "ReferenceClipped"
    REFERENCE_INFERENCE = "ReferenceInference"
    MKL_STYLE_SCALAR = "MklStyleScalar"
    VECTORIZED_SUM = "VectorizedSum"
    FULL_VECTORIZED = "FullVectorized"
    FULL_VECTORIZED_APPROX_EXP = "FullVectorizedApproxExp"

    @classmethod
    def from_name(cls, name: str) -> "KernelVariant":
        for v in cls:
            if v.value == name:
                return v
        raise ArgumentError(f"unknown variant {name!r}; choose from {[v.value for v in cls]}")


LADDER: tuple[KernelVariant, ...] = tuple(KernelVariant)

#: Floor applied to shifted logits by ReferenceClipped (kernels.py:99).
CLIP_FLOOR = np.float32(-64.0)
#: Smallest positive normal float32; results below it flush to +0.0 (kernels.py:101).
FLT_MIN_NORMAL = np.float32(1.1754943508222875e-38)

#: Fault-injection hook (kernels.py:103-105): when True the kernels shift by 0
#: instead of the row max, so large logits overflow exp and verification fails.
_SKIP_MAX_SHIFT = False


class RowStats(NamedTuple):
    """Per-row reduction results (kernels.py:108-112)."""

    max: Any
    sum: Any


def as_variant(variant) -> KernelVariant:
    """This package's KernelVariant for ``variant``: its own members, or the
    reference's own enum (softmax_kit.kernels.KernelVariant, kernels.py:76-93 --
    same member values), so a caller that swaps only the ``softmax`` import
    keeps passing its variants; anything else is an ArgumentError
    (kernels.py:304-305)."""
    if isinstance(variant, KernelVariant):
        return variant
    if isinstance(variant, enum.Enum) and isinstance(variant.value, str):
        for v in KernelVariant:
            if v.value == variant.value:
                return v
    raise ArgumentError(f"expected a KernelVariant, got {variant!r}")


def variant_mode(variant: KernelVariant) -> int:
    """Variant -> native arithmetic mode (include/softmax_b200.h, sk_mode)."""
    variant = as_variant(variant)
    if variant is KernelVariant.REFERENCE_CLIPPED:
        return _native.SK_MODE_CLIPPED
    if variant is KernelVariant.FULL_VECTORIZED_APPROX_EXP:
        return _native.SK_MODE_APPROX
    return _native.SK_MODE_EXACT


_hook_state = {"skip": False}
_hook_lock = threading.Lock()


def _sync_fault_hook() -> None:
    want = bool(_SKIP_MAX_SHIFT)
    if want != _hook_state["skip"]:
        with _hook_lock:
            _native.set_tuning("skip_max_shift", int(want))
            _hook_state["skip"] = want


def _check_cfg(cfg: LaneConfig) -> None:
    """This package's LaneConfig or the reference's (simd_reduce.py:60-75, a
    frozen dataclass with ``width``): same validation rule, no numeric effect."""
    if isinstance(cfg, LaneConfig):
        return
    w = getattr(cfg, "width", None)
    if isinstance(w, int) and not isinstance(w, bool):
        LaneConfig(w)  # same rule, same error
        return
    raise ArgumentError(f"expected a LaneConfig, got {cfg!r}")


def _is_foreign_matrix(m) -> bool:
    """A Matrix2D of another class with the reference's interface
    (tensor.py:31-72: rows, cols, a flat float32 ``data`` buffer, ``view2d``),
    e.g. softmax_kit.tensor.Matrix2D itself."""
    return (not isinstance(m, Matrix2D) and isinstance(getattr(m, "data", None), np.ndarray)
            and isinstance(getattr(m, "rows", None), (int, np.integer))
            and isinstance(getattr(m, "cols", None), (int, np.integer))
            and hasattr(type(m), "view2d"))


def _foreign_view(m, what: str) -> np.ndarray:
    """Validate a foreign Matrix2D like Matrix2D.__post_init__ (tensor.py:43-57)
    and return its (rows, cols) view."""
    rows, cols, data = int(m.rows), int(m.cols), m.data
    if rows < 1 or cols < 1:
        raise ArgumentError(f"matrix dimensions must be >= 1, got {rows}x{cols}")
    if data.dtype != np.float32:
        raise ArgumentError(f"expected float32 data, got {data.dtype}")
    if data.ndim != 1 or not data.flags.c_contiguous:
        raise ArgumentError("data must be a contiguous 1-D buffer")
    if data.size != rows * cols:
        raise ArgumentError(f"data length {data.size} != rows*cols = {rows * cols}")
    if what == "out" and not data.flags.writeable:
        raise ArgumentError("out must be writeable")
    return data.reshape(rows, cols)


def _foreign_error(m, e: Exception) -> Exception:
    """``e`` re-typed so the caller's own error classes catch it too: for a
    reference Matrix2D (softmax_kit.tensor) the raised class derives from both
    this package's class and softmax_kit.errors' class of the same name
    (errors.py:4-21), so ``except softmax_kit.errors.NumericDomainError`` works
    after swapping only the ``softmax`` import."""
    import sys

    mod = sys.modules.get(type(m).__module__.rsplit(".", 1)[0] + ".errors")
    theirs = getattr(mod, type(e).__name__, None) if mod else None
    if not (isinstance(theirs, type) and issubclass(theirs, Exception)) or isinstance(e, theirs):
        return e
    key = (type(e), theirs)
    cls = _FOREIGN_ERR.get(key)
    if cls is None:
        cls = type(type(e).__name__, (type(e), theirs), {"__module__": type(e).__module__})
        _FOREIGN_ERR[key] = cls
    return cls(*e.args)


_FOREIGN_ERR: dict = {}


def _fresh_out(rows: int, cols: int) -> Matrix2D:
    """The fresh output of a host call (kernels.py:358).  Every element is
    overwritten by the call, so a large result comes from hostpin's pool of
    recycled, page-locked blocks when one is free; otherwise alloc_matrix."""
    data = hostpin.pooled_output(rows * cols)
    if data is None:
        return alloc_matrix(rows, cols)
    return Matrix2D(rows=rows, cols=cols, data=data)


def _foreign_out(m):
    """A fresh output of the caller's own Matrix2D class (kernels.py:358 returns
    a fresh Matrix2D), backed by a 32-B aligned buffer."""
    data = _fresh_out(int(m.rows), int(m.cols)).data
    try:
        return type(m)(rows=int(m.rows), cols=int(m.cols), data=data)
    except Exception:  # noqa: BLE001 -- a class we cannot construct: ours
        return Matrix2D(rows=int(m.rows), cols=int(m.cols), data=data)


# ---------------------------------------------------------------- host path
def _softmax_host(x2d: np.ndarray, out2d: np.ndarray, mode: int, device: int) -> None:
    rows, cols = x2d.shape
    bad = ctypes.c_int64(-1)
    # a large caller buffer seen again is page-locked in place (hostpin.py):
    # the call below then DMAs straight from / into it, no staging copies
    hostpin.note(x2d)
    hostpin.note(out2d)
    st = _native.lib().sk_softmax_f32_host(
        x2d.ctypes.data, out2d.ctypes.data, rows, cols, mode, device, ctypes.byref(bad)
    )
    if st == _native.SK_ERR_NONFINITE:
        raise NumericDomainError(f"non-finite logits in row {bad.value}")  # kernels.py:347
    _native.check(st, "softmax")


# -------------------------------------------------------------- device path
_flags: dict[int, Any] = {}
_NULL_CTX = contextlib.nullcontext()


class _DeviceFlag:
    """The library's per-device non-finite flag (sk_device_flag): one device
    uint64 shared by every entry point on the device -- the Python wrappers
    here and the torch.ops launchers (torch_ops/sk_torch_ops.cpp) -- so a bad
    row recorded by an asynchronous call is raised by the next check.  Reads
    go through sk_flag_read on the device's current stream (like
    ``Tensor.item()``, they wait for it)."""

    def __init__(self, torch, index: int):
        self._torch, self.index = torch, index
        p = ctypes.c_void_p()
        _native.check(_native.lib().sk_device_flag(index, ctypes.byref(p)), "device_flag")
        self.ptr = int(p.value)

    def data_ptr(self) -> int:
        return self.ptr

    def _read(self, reset: int) -> int:
        v = ctypes.c_uint64()
        s = self._torch.cuda.current_stream(self.index).cuda_stream
        _native.check(_native.lib().sk_flag_read(self.ptr, s, reset, ctypes.byref(v)), "flag_read")
        return ctypes.c_int64(v.value).value  # SK_NO_BAD_ROW -> -1, aborted -> -2

    def item(self) -> int:
        return self._read(0)

    def fill_(self, value: int) -> "_DeviceFlag":
        if value != -1:
            raise ValueError("the device flag can only be cleared")
        self._read(1)
        return self


def _bad_flag(torch, device):
    idx = device.index if device.index is not None else torch.cuda.current_device()
    f = _flags.get(idx)
    if f is None:
        f = _DeviceFlag(torch, idx)
        _flags[idx] = f
    return f


def _torch():
    import torch  # plumbing only: device memory, streams

    return torch


def softmax_into(x, out, variant: KernelVariant, cfg: LaneConfig = LaneConfig(), *,
                 check_finite: bool = True, stream=None) -> None:
    """Device hot path: ``out[:] = softmax(x)`` for CUDA tensors, no allocation.

    With ``check_finite`` the call synchronises on the stream to raise
    ``NumericDomainError`` for non-finite rows, like the reference; without it
    the call is fully asynchronous (the flag is still recorded and raised by
    the next checked call on this device).
    """
    torch = _torch()
    mode = variant_mode(variant)
    _check_cfg(cfg)
    _sync_fault_hook()
    for name, t in (("input", x), ("output", out)):
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise ArgumentError(f"{name} must be a CUDA torch.Tensor")
        if t.dtype != torch.float32:
            raise ArgumentError(f"expected float32 {name}, got {t.dtype}")
        if t.dim() != 2:
            raise ArgumentError(f"{name} must be 2-D [rows, cols], got {t.dim()}-D")
        if t.shape[1] > 1 and t.stride(1) != 1:  # a single row too (x[0:1, ::2])
            raise ArgumentError(f"{name} must have unit column stride")
    if x.shape != out.shape:
        raise ArgumentError(f"shape mismatch {tuple(x.shape)} vs {tuple(out.shape)}")
    if x.device != out.device:
        raise ArgumentError("input and output must be on the same device")
    rows, cols = x.shape
    if cols < 1:
        raise ArgumentError(f"matrix dimensions must be >= 1, got {rows}x{cols}")
    if rows == 0:
        return
    ldx = x.stride(0) if rows > 1 else cols
    ldy = out.stride(0) if rows > 1 else cols
    dev = x.device
    # the C entry point plans for the CURRENT device: switch only when needed
    # (the context manager is a visible share of a small call's host cost)
    ctx = torch.cuda.device(dev) if dev.index != torch.cuda.current_device() else _NULL_CTX
    with ctx:
        s = stream if stream is not None else torch.cuda.current_stream(dev)
        flag = _bad_flag(torch, dev)
        st = _native.lib().sk_softmax_f32(
            x.data_ptr(), out.data_ptr(), rows, cols, ldx, ldy, mode, flag.ptr, None, 0,
            s.cuda_stream,
        )
        if st:
            _native.check(st, "softmax")
        if check_finite:
            bad = int(flag.item())  # syncs the current stream
            _raise_if_aborted(flag, bad)
            if bad != -1:
                flag.fill_(-1)
                raise NumericDomainError(f"non-finite logits in row {bad}")


def softmax(m, variant: KernelVariant, cfg: LaneConfig = LaneConfig(), *,
            out=None, device: int | None = None, check_finite: bool = True):
    """Run one softmax variant over ``m`` and return a fresh output
    (kernels.py:350-362).  See the module docstring for accepted types."""
    if _is_foreign_matrix(m):
        try:
            return _softmax_matrix(m, variant, cfg, out, device)
        except SoftmaxKitError as e:
            raise _foreign_error(m, e) from None
    mode = variant_mode(variant)
    _check_cfg(cfg)
    _sync_fault_hook()
    if isinstance(m, Matrix2D):
        return _softmax_matrix(m, variant, cfg, out, device)
    if isinstance(m, np.ndarray):
        if m.ndim != 2 or m.dtype != np.float32:
            raise ArgumentError("numpy input must be a 2-D float32 array")
        if m.shape[0] < 1 or m.shape[1] < 1:
            raise ArgumentError(f"matrix dimensions must be >= 1, got {m.shape[0]}x{m.shape[1]}")
        x = np.ascontiguousarray(m)
        y = np.empty_like(x) if out is None else out
        if y.shape != x.shape or y.dtype != np.float32 or not y.flags.c_contiguous:
            raise ArgumentError("out must be a C-contiguous float32 array of the input's shape")
        _softmax_host(x, y, mode, _host_device(device))
        return y
    torch = _torch()
    if isinstance(m, torch.Tensor):
        if not m.is_cuda:
            raise ArgumentError("torch input must be a CUDA tensor (there is no CPU path)")
        y = torch.empty(m.shape, dtype=torch.float32, device=m.device) if out is None else out
        softmax_into(m, y, variant, cfg, check_finite=check_finite)
        return y
    raise ArgumentError(f"unsupported input type {type(m).__name__}")


def _softmax_matrix(m, variant, cfg, out, device):
    """The host-buffer path for this package's or a foreign Matrix2D."""
    mode = variant_mode(variant)
    _check_cfg(cfg)
    _sync_fault_hook()
    x2d = m.view2d if isinstance(m, Matrix2D) else _foreign_view(m, "input")
    if out is None:
        out = _fresh_out(m.rows, m.cols) if isinstance(m, Matrix2D) else _foreign_out(m)
    if isinstance(out, Matrix2D):
        y2d = out.view2d
    elif _is_foreign_matrix(out):
        y2d = _foreign_view(out, "out")
    else:
        raise ArgumentError("out must be a Matrix2D of the input's shape")
    if y2d.shape != x2d.shape:
        raise ArgumentError("out must be a Matrix2D of the input's shape")
    _softmax_host(x2d, y2d, mode, _host_device(device))
    return out


def _host_device(device: int | None) -> int:
    if device is not None:
        return int(device)
    try:
        torch = _torch()
        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:  # pragma: no cover - torch import problems surface below
        pass
    return 0


def row_stats_device(x, variant: KernelVariant = KernelVariant.REFERENCE_CLIPPED):
    """Per-row (max, sum of exp(clip(x - max))) of a CUDA [N, C] tensor -- the
    RowStats pair (kernels.py:108-112, 272-276) the column shard exchanges.
    Returns ``RowStats(max=float32[N], sum=float64[N])`` CUDA tensors."""
    torch = _torch()
    mode = variant_mode(variant)
    _sync_fault_hook()
    if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype != torch.float32 or x.dim() != 2:
        raise ArgumentError("x must be a 2-D float32 CUDA tensor")
    if x.shape[1] > 1 and x.stride(1) != 1:
        raise ArgumentError("x must have unit column stride")
    rows, cols = x.shape
    if cols < 1:
        raise ArgumentError("cols must be >= 1")
    rmax = torch.empty(rows, dtype=torch.float32, device=x.device)
    rsum = torch.empty(rows, dtype=torch.float64, device=x.device)
    if rows:
        with torch.cuda.device(x.device):
            flag = _bad_flag(torch, x.device)
            _native.check(
                _native.lib().sk_row_stats_f32(
                    x.data_ptr(), rows, cols, x.stride(0) if rows > 1 else cols, mode,
                    rmax.data_ptr(), rsum.data_ptr(), flag.data_ptr(), None, 0,
                    torch.cuda.current_stream(x.device).cuda_stream),
                "row_stats",
            )
    return RowStats(max=rmax, sum=rsum)


EXCHANGE_ABORTED = -2  # SK_EXCHANGE_ABORTED as int64


def _raise_if_aborted(flag, bad: int) -> None:
    if bad == EXCHANGE_ABORTED:
        flag.fill_(-1)
        raise SoftmaxKitError("row-statistics exchange timed out (a peer never arrived)")


def check_device_flag(device=None) -> None:
    """Raise NumericDomainError if an unchecked call on ``device`` saw bad rows."""
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    flag = _bad_flag(torch, dev)
    bad = int(flag.item())
    _raise_if_aborted(flag, bad)
    if bad != -1:
        flag.fill_(-1)
        raise NumericDomainError(f"non-finite logits in row {bad}")


def _require_cuda() -> None:
    torch = _torch()
    if not torch.cuda.is_available():
        raise SoftmaxKitError("no CUDA device: this package has no CPU fallback")
