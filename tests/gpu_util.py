"""Helpers for GPU tests: call the C ABI directly on torch device memory."""

from __future__ import annotations

import numpy as np

from paper_1904_12380_b200 import _native

NO_BAD = -1


def torch():
    import torch as t

    return t


def to_dev(x: np.ndarray, offset: int = 0, ld: int | None = None):
    """Copy a 2-D float32 array to the GPU, optionally at a float offset from
    a 256-B aligned base and/or with row pitch ``ld`` (elements)."""
    t = torch()
    rows, cols = x.shape
    ld = ld or cols
    buf = t.full((offset + rows * ld + 8,), float("nan"), dtype=t.float32, device="cuda")
    view = buf[offset:offset + rows * ld].view(rows, ld)[:, :cols]
    view.copy_(t.from_numpy(np.ascontiguousarray(x)))
    return buf, view


def softmax_abi(x: np.ndarray, mode: int = 0, x_offset: int = 0, y_offset: int = 0,
                ldx: int | None = None, ldy: int | None = None, expect_bad: bool = False):
    """Run sk_softmax_f32 on a copy of ``x``; returns (y numpy, bad_row)."""
    t = torch()
    rows, cols = x.shape
    ldx = ldx or cols
    ldy = ldy or cols
    _, xd = to_dev(x, x_offset, ldx)
    ybuf = t.full((y_offset + rows * ldy + 8,), float("nan"), dtype=t.float32, device="cuda")
    yd = ybuf[y_offset:y_offset + rows * ldy].view(rows, ldy)[:, :cols]
    flag = t.full((1,), -1, dtype=t.int64, device="cuda")
    st = _native.lib().sk_softmax_f32(
        xd.data_ptr(), yd.data_ptr(), rows, cols, ldx, ldy, mode, flag.data_ptr(), None, 0,
        t.cuda.current_stream().cuda_stream)
    _native.check(st, "sk_softmax_f32")
    t.cuda.synchronize()
    bad = int(flag.item())
    y = yd.cpu().numpy().copy()
    # pitch padding must be untouched
    if ldy > cols and rows:
        pad = ybuf[y_offset:y_offset + rows * ldy].view(rows, ldy)[:, cols:]
        assert t.isnan(pad).all(), "kernel wrote outside [rows, cols]"
    return y, bad


def plan(rows: int, cols: int) -> str:
    return _native.describe_plan(rows, cols, cols, cols, 0, 0, 0)


def parity_all_rows(oracle, y_dev, x_host: np.ndarray, chunk_bytes: int = 64 << 20) -> dict:
    """Every row of a device output against the oracle, in row chunks (so the
    full c4 / c5a / c5b outputs fit host memory); worst metrics + gate."""
    rows, cols = x_host.shape
    step = max(1, chunk_bytes // (4 * cols))
    worst = {"max_abs": 0.0, "max_rel": 0.0, "max_rowsum_dev": 0.0}
    for a in range(0, rows, step):
        b = min(rows, a + step)
        ref = oracle.softmax_ref(x_host[a:b], True, nthreads=0)
        d = oracle.parity(y_dev[a:b].cpu().numpy(), ref)
        for k in worst:
            worst[k] = max(worst[k], d[k])
    worst["ok"] = bool(worst["max_abs"] <= oracle.TOL_ABS and worst["max_rel"] <= oracle.TOL_REL
                       and worst["max_rowsum_dev"] <= oracle.TOL_ROWSUM)
    worst["rows_checked"] = rows
    return worst
