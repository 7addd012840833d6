"""CPU oracle for the row-softmax hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module; the product package
(paper_1904_12380_b200/) never does.

``libsk_oracle.so`` (oracle/sk_oracle.c) is a plain-C restatement of the
reference's ReferenceClipped / ReferenceInference pipeline
(/root/reference/pkg/src/softmax_kit/kernels.py:136-189, 342-362).  It is
pinned bit-for-bit against the reference itself: tests/golden/make_golden.py
imports the reference package in the build container, runs it, and commits
its outputs and output hashes (tests/golden/golden.npz, golden.json);
tests/test_oracle_golden.py checks this oracle against them.

The error metrics restate oracle.py:52-69 of the reference.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import c_double, c_float, c_int, c_int64, c_uint64, c_void_p
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libsk_oracle.so"
_lib = None


def build(force: bool = False) -> Path:
    """gcc the C restatement into libsk_oracle.so next to it (test
    infrastructure; self-contained so that loading the checker never imports
    the product package or maps its library)."""
    import subprocess

    src = HERE / "sk_oracle.c"
    if not force and LIB_PATH.exists() and LIB_PATH.stat().st_mtime >= src.stat().st_mtime:
        return LIB_PATH
    tmp = LIB_PATH.with_suffix(".so.tmp")
    # -O2, no -ffast-math: the f64 left-to-right sum and IEEE reciprocal are the contract.
    cmd = ["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-std=c11", str(src), "-o", str(tmp),
           "-lm"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed: {' '.join(cmd)}\n{r.stdout}{r.stderr}")
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()  # no-op unless missing or older than sk_oracle.c
        L = ctypes.CDLL(str(LIB_PATH))
        L.sko_softmax_f32.restype = c_int64
        L.sko_softmax_f32.argtypes = [c_void_p, c_void_p, c_int64, c_int64, c_int, c_int]
        L.sko_pipeline_f32.restype = None
        L.sko_pipeline_f32.argtypes = [c_void_p, c_void_p, c_int64, c_int64, c_int, c_int]
        L.sko_first_nonfinite_row.restype = c_int64
        L.sko_first_nonfinite_row.argtypes = [c_void_p, c_int64, c_int64]
        L.sko_lanes_max.restype = c_float
        L.sko_lanes_max.argtypes = [c_void_p, c_int64, c_int]
        L.sko_lanes_sum.restype = c_float
        L.sko_lanes_sum.argtypes = [c_void_p, c_int64, c_int]
        L.sko_philox_raw.restype = None
        L.sko_philox_raw.argtypes = [c_uint64, c_uint64, c_void_p, c_int64]
        L.sko_max_threads.restype = c_int
        L.sko_seq_max.restype = c_float
        L.sko_seq_max.argtypes = [c_void_p, c_int64]
        L.sko_seq_sum_wide.restype = c_float
        L.sko_seq_sum_wide.argtypes = [c_void_p, c_int64]
        L.sko_fill_uniform_f32.restype = None
        L.sko_fill_uniform_f32.argtypes = [c_void_p, c_int64, c_uint64, c_double, c_double,
                                           c_uint64, c_int]
        L.sko_fill_normal_f32.restype = None
        L.sko_fill_normal_f32.argtypes = [c_void_p, c_int64, c_uint64, c_double, c_uint64, c_int]
        L.sko_plant_f32.restype = c_int
        L.sko_plant_f32.argtypes = [c_void_p, c_int64, c_int64, c_uint64, c_float]
        _lib = L
    return _lib


def max_threads() -> int:
    return int(lib().sko_max_threads())


def _c2d(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    if x.ndim != 2:
        raise ValueError("expected a 2-D array")
    return x


def softmax_ref(x: np.ndarray, clip: bool = True, nthreads: int = 1,
                out: np.ndarray | None = None) -> np.ndarray:
    """ReferenceClipped (clip=True) / ReferenceInference (clip=False) softmax.

    Raises ValueError("non-finite logits in row r") like kernels.py:342-347.
    """
    x = _c2d(x)
    y = np.empty_like(x) if out is None else out
    bad = lib().sko_softmax_f32(x.ctypes.data, y.ctypes.data, x.shape[0], x.shape[1],
                                int(clip), nthreads)
    if bad >= 0:
        raise ValueError(f"non-finite logits in row {bad}")
    return y


def pipeline(x: np.ndarray, y: np.ndarray, clip: bool = True, nthreads: int = 1) -> None:
    """maxsub -> exp -> sumscale without the finite scan (profiler.py:136-162 timing)."""
    lib().sko_pipeline_f32(x.ctypes.data, y.ctypes.data, x.shape[0], x.shape[1], int(clip),
                           nthreads)


def first_nonfinite_row(x: np.ndarray) -> int:
    x = _c2d(x)
    return int(lib().sko_first_nonfinite_row(x.ctypes.data, x.shape[0], x.shape[1]))


def lanes_max(a: np.ndarray, W: int) -> np.float32:
    a = np.ascontiguousarray(a, dtype=np.float32)
    return np.float32(lib().sko_lanes_max(a.ctypes.data, a.size, W))


def lanes_sum(a: np.ndarray, W: int) -> np.float32:
    a = np.ascontiguousarray(a, dtype=np.float32)
    return np.float32(lib().sko_lanes_sum(a.ctypes.data, a.size, W))


# ---- the 1-D component operations (reference kernels.py:229-276) -----------
# Restated with the same arithmetic: strict scans in C, IEEE fp32 elementwise
# ops in numpy, and numpy's own exp for exp_batch / row_stats (the reference
# calls np.exp there: kernels.py:254, 275).
def _row(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    if a.ndim != 1 or a.size == 0:
        raise ValueError("expected a non-empty 1-D row")
    return a


def row_max_scalar(a) -> np.float32:
    a = _row(a)
    return np.float32(lib().sko_seq_max(a.ctypes.data, a.size))


def subtract_broadcast(a, v: float) -> np.ndarray:
    return _row(a) - np.float32(v)


def value_clip(x: float) -> np.float32:
    x32 = np.float32(x)
    return x32 if x32 > np.float32(-64.0) else np.float32(-64.0)


def exp_batch(a) -> np.ndarray:
    return np.exp(np.asarray(a, dtype=np.float32))


def row_sum_scalar(a) -> np.float32:
    a = _row(a)
    return np.float32(lib().sko_seq_sum_wide(a.ctypes.data, a.size))


def scale_reciprocal(a, s: float) -> np.ndarray:
    return _row(a) * (np.float32(1.0) / np.float32(s))


def row_stats(a) -> tuple[np.float32, np.float32]:
    m = row_max_scalar(a)
    return m, row_sum_scalar(np.exp(subtract_broadcast(a, m)))


def philox_raw(seed: int, start: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.uint64)
    lib().sko_philox_raw(seed, start, out.ctypes.data, n)
    return out


# ---- error metrics (reference oracle.py:52-69, plus max |abs|) -------------
def max_abs_err(got: np.ndarray, ref: np.ndarray) -> float:
    g = np.asarray(got, dtype=np.float64)
    if not np.isfinite(g).all():
        return float("inf")
    return float(np.max(np.abs(g - np.asarray(ref, dtype=np.float64)))) if g.size else 0.0


#: the flush threshold of the unclipped rungs (kernels.py:101, :186-188)
FLT_MIN_NORMAL = 1.1754943508222875e-38


def max_rel_err(got: np.ndarray, ref: np.ndarray) -> float:
    """Largest |got - ref| / |ref| over ref != 0; inf if got is non-finite or
    differs from an exact-zero reference (oracle.py:52-61 assumes ref > 0,
    which the clip guarantees; unclipped references may hold exact zeros).

    Flush boundary: the unclipped rungs flush y < FLT_MIN to +0, so a value
    within the relative tolerance of FLT_MIN may legitimately land on either
    side.  A zero against a value <= FLT_MIN * (1 + 1e-5) counts as a match;
    any other zero / non-zero disagreement is inf."""
    g = np.asarray(got, dtype=np.float64)
    r = np.asarray(ref, dtype=np.float64)
    if not np.isfinite(g).all():
        return float("inf")
    if g.size == 0:
        return 0.0
    edge = FLT_MIN_NORMAL * (1.0 + 1e-5)
    flip = ((r == 0) & (g != 0) & (np.abs(g) <= edge)) | ((g == 0) & (r != 0) & (np.abs(r) <= edge))
    if flip.any():
        g = np.where(flip, 0.0, g)
        r = np.where(flip, 0.0, r)
    nz = r != 0
    if np.any(g[~nz] != 0):
        return float("inf")
    if not nz.any():
        return 0.0
    return float(np.max(np.abs(g[nz] - r[nz]) / np.abs(r[nz])))


def max_rowsum_dev(got: np.ndarray) -> float:
    g = np.asarray(got, dtype=np.float64)
    if not np.isfinite(g).all():
        return float("inf")
    return float(np.max(np.abs(g.sum(axis=1) - 1.0))) if g.size else 0.0


#: North-star parity gate vs ReferenceClipped on identical inputs
#: (BASELINE.json north_star).
TOL_ABS = 1e-6
TOL_REL = 1e-5
TOL_ROWSUM = 1e-5
#: FullVectorizedApproxExp tolerance (reference bench.py:52).
TOL_REL_APPROX = 1e-5


def parity(got: np.ndarray, ref: np.ndarray, approx: bool = False) -> dict:
    d = {
        "max_abs": max_abs_err(got, ref),
        "max_rel": max_rel_err(got, ref),
        "max_rowsum_dev": max_rowsum_dev(got),
    }
    tol_rel = TOL_REL_APPROX if approx else TOL_REL
    d["ok"] = bool(d["max_abs"] <= TOL_ABS or approx) and d["max_rel"] <= tol_rel and \
        d["max_rowsum_dev"] <= TOL_ROWSUM
    return d


def cpu_count() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
