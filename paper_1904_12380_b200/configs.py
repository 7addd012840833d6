"""The BASELINE.json workloads as seeded synthetic inputs.

BASELINE.json names no public dataset; each config is a fixed seeded
generator with the stated shape and distribution:

  c1  [4096, 50]        N(0, 4^2), seed 0        (DAM-attention-like)
  c2  [65536, 128]      U(-10, 10), seed 1       (reference fill_uniform, tensor.py:106-121)
  c3  [8192, 1000]      N(0, 3^2), seed 2, 1% of positions (81,920) set to -100
  c4  [512, 262144]     N(0, 5^2), seed 3
  c5a [2097152, 256]    N(0, 1), seed 4          (row-sharded across GPUs)
  c5b [1024, 1048576]   N(0, 2^2), seed 5        (column-sharded across GPUs)

Element i of a config depends only on (seed, i), so any row range can be
generated on its own (each rank generates its shard of the same global
matrix) -- except c3's planted positions, which need the whole matrix.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

from .errors import ArgumentError
from .tensor import fill_normal_array, fill_uniform_array, plant_value


@dataclass(frozen=True)
class InputSpec:
    name: str
    rows: int
    cols: int
    dist: str  # "normal" | "uniform"
    seed: int
    sigma: float = 1.0
    low: float = 0.0
    high: float = 1.0
    plant_count: int = 0
    plant_value: float = 0.0
    note: str = ""

    @property
    def elements(self) -> int:
        return self.rows * self.cols

    @property
    def bytes_io(self) -> int:
        """Algorithmic HBM bytes of one softmax: one fp32 read + one fp32 write."""
        return 8 * self.elements

    def describe(self) -> str:
        d = (f"N(0,{self.sigma:g}^2)" if self.dist == "normal"
             else f"U({self.low:g},{self.high:g})")
        s = f"{self.name} [{self.rows},{self.cols}] {d} seed {self.seed}"
        if self.plant_count:
            s += f", {self.plant_count} seeded positions = {self.plant_value:g}"
        return s


CONFIGS: dict[str, InputSpec] = {
    "c1": InputSpec("c1", 4096, 50, "normal", 0, sigma=4.0, note="DAM-attention-like"),
    "c2": InputSpec("c2", 65536, 128, "uniform", 1, low=-10.0, high=10.0,
                    note="short-row batch, warp-per-row"),
    "c3": InputSpec("c3", 8192, 1000, "normal", 2, sigma=3.0, plant_count=81920,
                    plant_value=-100.0, note="classifier width, ValueClip exercised"),
    "c4": InputSpec("c4", 512, 262144, "normal", 3, sigma=5.0, note="vocab-width long rows"),
    "c5a": InputSpec("c5a", 2097152, 256, "normal", 4, sigma=1.0, note="row-sharded scale"),
    "c5b": InputSpec("c5b", 1024, 1048576, "normal", 5, sigma=2.0, note="column-sharded scale"),
}


def get(name: str) -> InputSpec:
    try:
        return CONFIGS[name]
    except KeyError:
        raise ArgumentError(f"unknown config {name!r}; choose from {sorted(CONFIGS)}") from None


def generate(spec: InputSpec | str, row_start: int = 0, row_count: int | None = None,
             out: np.ndarray | None = None, nthreads: int = 0) -> np.ndarray:
    """Rows ``[row_start, row_start + row_count)`` of the config as a 2-D
    float32 array (``out`` may be any C-contiguous float32 buffer of that size,
    e.g. a pinned Matrix2D view)."""
    if isinstance(spec, str):
        spec = get(spec)
    if row_count is None:
        row_count = spec.rows - row_start
    if row_start < 0 or row_count < 0 or row_start + row_count > spec.rows:
        raise ArgumentError("row range outside the config")
    if spec.plant_count and (row_start != 0 or row_count != spec.rows):
        raise ArgumentError(f"{spec.name}: planted positions need the whole matrix")
    shape = (row_count, spec.cols)
    if out is None:
        out = np.empty(shape, dtype=np.float32)
    out = out.reshape(shape)
    start = row_start * spec.cols
    if spec.dist == "normal":
        fill_normal_array(out, spec.seed, spec.sigma, start, nthreads)
    elif spec.dist == "uniform":
        fill_uniform_array(out, spec.seed, spec.low, spec.high, start, nthreads)
    else:  # pragma: no cover
        raise ArgumentError(f"unknown distribution {spec.dist}")
    if spec.plant_count:
        plant_value(out, spec.plant_count, spec.seed, spec.plant_value)
    return out


def generate_cols(spec: InputSpec | str, col_start: int, col_count: int,
                  out: np.ndarray | None = None, nthreads: int = 0) -> np.ndarray:
    """Columns ``[col_start, col_start + col_count)`` of every row of the config
    (a column shard: rank r of N owns columns [r*C/N, (r+1)*C/N)); element
    (r, c) is element r*C + c of the config's stream, as in ``generate``."""
    if isinstance(spec, str):
        spec = get(spec)
    if spec.plant_count:
        raise ArgumentError(f"{spec.name}: planted positions need the whole matrix")
    if col_start < 0 or col_count < 0 or col_start + col_count > spec.cols:
        raise ArgumentError("column range outside the config")
    if out is None:
        out = np.empty((spec.rows, col_count), dtype=np.float32)
    out = out.reshape(spec.rows, col_count)
    for r in range(spec.rows):
        start = r * spec.cols + col_start
        if spec.dist == "normal":
            fill_normal_array(out[r], spec.seed, spec.sigma, start, nthreads)
        else:
            fill_uniform_array(out[r], spec.seed, spec.low, spec.high, start, nthreads)
    return out


def generate_rows_extended(spec: InputSpec | str, row_start: int, row_count: int,
                           out: np.ndarray | None = None, nthreads: int = 0) -> np.ndarray:
    """Rows of the config's stream beyond ``spec.rows`` (weak scaling: rank r
    of N owns rows [r*rows, (r+1)*rows) of an N*rows global matrix)."""
    if isinstance(spec, str):
        spec = get(spec)
    if spec.plant_count:
        raise ArgumentError(f"{spec.name}: planted configs cannot be extended")
    big = InputSpec(spec.name, max(spec.rows, row_start + row_count), spec.cols, spec.dist,
                    spec.seed, spec.sigma, spec.low, spec.high)
    return generate(big, row_start, row_count, out, nthreads)


def sha256(a: np.ndarray) -> str:
    """Input hash recorded next to every result (bench.py:115-119)."""
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8).reshape(-1).data).hexdigest()
