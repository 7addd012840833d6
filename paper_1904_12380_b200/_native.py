"""ctypes binding of the C ABI (include/softmax_b200.h).

This is the binding a maintainer of the reference would add:
plain pointers, sizes and a stream handle.  There is no fallback: if the
shared library is missing, importing the compute entry points raises.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_int64, c_size_t, c_uint64, c_void_p
from pathlib import Path

from .errors import ArgumentError, NumericDomainError, ResourceError, SoftmaxKitError

# SK_LIB_PATH: load another build of this library (A/B timing of two builds)
LIB_PATH = Path(os.environ.get("SK_LIB_PATH") or
                Path(__file__).resolve().with_name("libsoftmax_b200.so"))

SK_OK = 0
SK_ERR_ARGUMENT = 1
SK_ERR_NONFINITE = 2
SK_ERR_CUDA = 3
SK_ERR_RESOURCE = 4

SK_MODE_CLIPPED = 0
SK_MODE_EXACT = 1
SK_MODE_APPROX = 2

SK_NO_BAD_ROW = 0xFFFFFFFFFFFFFFFF

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None

# name -> (restype, argtypes); every function declared in include/softmax_b200.h
SIGNATURES: dict[str, tuple] = {
    "sk_abi_version": (c_int, []),
    "sk_status_string": (c_char_p, [c_int]),
    "sk_last_error": (c_char_p, []),
    "sk_softmax_f32": (
        c_int,
        [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64, c_int, c_void_p, c_void_p,
         c_size_t, c_void_p],
    ),
    "sk_softmax_workspace_bytes": (c_size_t, [c_int64, c_int64]),
    "sk_softmax_f32_host": (
        c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int, c_int, POINTER(c_int64)]
    ),
    "sk_row_stats_f32": (
        c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_int, c_void_p, c_void_p, c_void_p, c_void_p,
         c_size_t, c_void_p],
    ),
    "sk_row_stats_workspace_bytes": (c_size_t, [c_int64, c_int64]),
    "sk_rescale_sumexp": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
    "sk_normalize_f32": (
        c_int,
        [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64, c_int, c_void_p, c_void_p,
         c_void_p],
    ),
    "sk_maxsub_f32": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64, c_int,
                              c_void_p]),
    "sk_exp_f32": (c_int, [c_void_p, c_int64, c_int, c_void_p]),
    "sk_sumscale_f32": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p]),
    "sk_row_sum_f32": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p]),
    "sk_row_stats_ref_f32": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "sk_shift_scale_f32": (c_int, [c_void_p, c_void_p, c_int64, c_float, c_float, c_void_p]),
    "sk_alloc_pinned": (c_void_p, [c_size_t]),
    "sk_free_pinned": (None, [c_void_p]),
    "sk_host_register": (c_int, [c_void_p, c_size_t]),
    "sk_host_unregister": (c_int, [c_void_p]),
    "sk_set_tuning": (c_int, [c_char_p, c_int]),
    "sk_copy_f32": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_void_p]),
    "sk_exp_accuracy": (c_int, [c_int, c_float, c_float, POINTER(c_double), POINTER(c_double), c_int]),
    "sk_describe_plan": (
        c_int, [c_int64, c_int64, c_int64, c_int64, c_uint64, c_uint64, c_int, c_char_p, c_int]
    ),
    "sk_fill_uniform_f32": (c_int, [c_void_p, c_int64, c_uint64, c_double, c_double, c_uint64, c_int]),
    "sk_fill_normal_f32": (c_int, [c_void_p, c_int64, c_uint64, c_double, c_uint64, c_int]),
    "sk_plant_f32": (c_int, [c_void_p, c_int64, c_int64, c_uint64, c_float]),
    "sk_xchg_block_bytes": (c_size_t, []),
    "sk_xchg_alloc": (c_int, [c_int, POINTER(c_void_p)]),
    "sk_xchg_free": (c_int, [c_void_p]),
    "sk_xchg_reset": (c_int, [c_void_p, c_void_p]),
    "sk_device_flag": (c_int, [c_int, POINTER(c_void_p)]),
    "sk_flag_read": (c_int, [c_void_p, c_void_p, c_int, POINTER(c_uint64)]),
    "sk_xchg_reset_period": (c_uint64, []),
    "sk_ipc_handle": (c_int, [c_void_p, c_void_p]),
    "sk_ipc_open": (c_int, [c_void_p, POINTER(c_void_p)]),
    "sk_ipc_close": (c_int, [c_void_p]),
    "sk_colshard_softmax_f32": (
        c_int,
        [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64, c_int, c_int, c_int, c_void_p,
         c_void_p, c_void_p],
    ),
    "sk_colshard_emulate_f32": (
        c_int,
        [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64, c_int, c_int, c_void_p, c_void_p,
         c_void_p],
    ),
    "sk_describe_colshard_plan": (c_int, [c_int64, c_int64, c_int, c_int, c_int, c_char_p, c_int]),
}

SK_IPC_HANDLE_BYTES = 64
SK_EXCHANGE_ABORTED = 0xFFFFFFFFFFFFFFFE


def lib() -> ctypes.CDLL:
    """Load libsoftmax_b200.so once; raise loudly if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback)"
                )
            L = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            # SK_TUNING="key=value key=value": tuning overrides at load (A/B runs)
            for kv in os.environ.get("SK_TUNING", "").split():
                k, _, v = kv.partition("=")
                if L.sk_set_tuning(k.encode(), int(v)) != 0:
                    raise ValueError(f"SK_TUNING: bad entry {kv!r}")
            _lib = L
    return _lib


def last_error() -> str:
    return (lib().sk_last_error() or b"").decode(errors="replace")


def check(status: int, what: str = "") -> None:
    """Map an sk_status onto the reference error taxonomy."""
    if status == SK_OK:
        return
    msg = last_error() or lib().sk_status_string(status).decode()
    if what:
        msg = f"{what}: {msg}"
    if status == SK_ERR_ARGUMENT:
        raise ArgumentError(msg)
    if status == SK_ERR_NONFINITE:
        raise NumericDomainError(msg)
    if status == SK_ERR_RESOURCE:
        raise ResourceError(msg)
    raise SoftmaxKitError(msg)


def set_tuning(key: str, value: int) -> None:
    check(lib().sk_set_tuning(key.encode(), int(value)), f"sk_set_tuning({key})")


def describe_colshard_plan(rows: int, cols: int, world: int, emulate: bool = False,
                           device: int = 0) -> str:
    buf = ctypes.create_string_buffer(256)
    check(lib().sk_describe_colshard_plan(rows, cols, world, 1 if emulate else 0, device, buf, 256))
    return buf.value.decode()


def describe_plan(rows: int, cols: int, ldx: int | None = None, ldy: int | None = None,
                  x_addr: int = 0, y_addr: int = 0, device: int = 0) -> str:
    buf = ctypes.create_string_buffer(256)
    check(lib().sk_describe_plan(rows, cols, ldx or cols, ldy or cols, x_addr, y_addr, device,
                                 buf, 256))
    return buf.value.decode()
