"""Randomised differential test: the C ABI against the oracle on seeded random
shapes that sweep every planner path (K1 shapes, K1 medium rows, K1m 128/32-bit,
K3g aligned / unaligned, the latency path, K3c, K4) with random base offsets,
row pitches, modes and value scales -- plus the host-buffer path."""

import numpy as np
import pytest

import paper_1904_12380_b200 as sk
from paper_1904_12380_b200 import tensor
from tests import gpu_util as gu

pytestmark = pytest.mark.gpu

MAX_ELEMS = 3_000_000


def _case(rng):
    cols = int(np.exp(rng.uniform(0.0, np.log(300_000))))
    cols = max(1, cols + int(rng.integers(-3, 4)))
    if rng.random() < 0.5:
        cols = max(4, cols // 4 * 4)  # half the cases 128-bit friendly
    rows = int(rng.integers(1, max(2, min(700, MAX_ELEMS // cols) + 1)))
    xo = int(rng.integers(0, 4)) if rng.random() < 0.3 else 0
    yo = int(rng.integers(0, 4)) if rng.random() < 0.3 else 0
    ldx = cols + (int(rng.integers(0, 8)) if rng.random() < 0.3 else 0)
    ldy = cols + (int(rng.integers(0, 8)) if rng.random() < 0.3 else 0)
    mode = int(rng.choice([0, 0, 1, 2]))
    sigma = float(rng.choice([0.1, 3.0, 30.0]))
    return rows, cols, xo, yo, ldx, ldy, mode, sigma


@pytest.mark.parametrize("seed", range(12))
def test_random_shapes_against_oracle(seed, oracle):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(12):
        rows, cols, xo, yo, ldx, ldy, mode, sigma = _case(rng)
        x = np.empty((rows, cols), np.float32)
        tensor.fill_normal_array(x, int(rng.integers(0, 1 << 30)), sigma)
        if rng.random() < 0.3:  # a dominant logit and a clipped one
            x[int(rng.integers(0, rows)), int(rng.integers(0, cols))] += 80.0
            x[int(rng.integers(0, rows)), int(rng.integers(0, cols))] -= 400.0
        y, bad = gu.softmax_abi(x, mode, x_offset=xo, y_offset=yo, ldx=ldx, ldy=ldy)
        what = (rows, cols, xo, yo, ldx, ldy, mode, sigma, gu.plan(rows, cols))
        assert bad == gu.NO_BAD, what
        d = oracle.parity(y, oracle.softmax_ref(x, clip=(mode == 0)), approx=(mode == 2))
        assert d["ok"], (what, d)


def _short_case(rng):
    """Short / medium rows (K1's 128-, 64- and 32-bit shapes, exact-fit NV,
    job-size variants): offsets of 0-3 floats give 16-, 8- and 4-B bases."""
    cols = int(rng.integers(1, 3073)) if rng.random() < 0.5 else int(rng.integers(1, 300))
    if rng.random() < 0.3:
        cols = max(2, cols // 2 * 2)  # even rows: the 64-bit path when 8-B aligned
    elems = int(np.exp(rng.uniform(np.log(cols), np.log(MAX_ELEMS))))
    rows = max(1, elems // cols)
    xo = int(rng.integers(0, 4)) if rng.random() < 0.4 else 0
    yo = xo if rng.random() < 0.7 else int(rng.integers(0, 4))
    ldx = cols + (int(rng.integers(0, 4)) if rng.random() < 0.3 else 0)
    ldy = cols + (int(rng.integers(0, 4)) if rng.random() < 0.3 else 0)
    mode = int(rng.choice([0, 0, 1, 2]))
    sigma = float(rng.choice([0.1, 3.0, 30.0]))
    return rows, cols, xo, yo, ldx, ldy, mode, sigma


@pytest.mark.parametrize("seed", range(8))
def test_random_short_rows_against_oracle(seed, oracle):
    rng = np.random.default_rng(3000 + seed)
    for _ in range(10):
        rows, cols, xo, yo, ldx, ldy, mode, sigma = _short_case(rng)
        x = np.empty((rows, cols), np.float32)
        tensor.fill_normal_array(x, int(rng.integers(0, 1 << 30)), sigma)
        if rng.random() < 0.3:
            x[int(rng.integers(0, rows)), int(rng.integers(0, cols))] += 80.0
            x[int(rng.integers(0, rows)), int(rng.integers(0, cols))] -= 400.0
        y, bad = gu.softmax_abi(x, mode, x_offset=xo, y_offset=yo, ldx=ldx, ldy=ldy)
        what = (rows, cols, xo, yo, ldx, ldy, mode, sigma, gu.plan(rows, cols))
        assert bad == gu.NO_BAD, what
        idx = np.unique(np.r_[0:min(rows, 3000), max(0, rows - 3000):rows])
        d = oracle.parity(y[idx], oracle.softmax_ref(x[idx], clip=(mode == 0)), approx=(mode == 2))
        assert d["ok"], (what, d)
        assert np.isfinite(y).all() and (y >= 0).all(), what


@pytest.mark.parametrize("seed", range(3))
def test_random_shapes_host_path(seed, oracle):
    rng = np.random.default_rng(2000 + seed)
    for _ in range(6):
        rows, cols, *_ = _case(rng)
        x = np.empty((rows, cols), np.float32)
        tensor.fill_normal_array(x, seed * 100 + cols, 4.0)
        out = sk.softmax(sk.Matrix2D.from_array(x, pinned=bool(rng.random() < 0.5)),
                         sk.KernelVariant.REFERENCE_CLIPPED)
        d = oracle.parity(out.view2d, oracle.softmax_ref(x))
        assert d["ok"], (rows, cols, d)
