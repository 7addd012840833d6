"""The BASELINE.json configs as seeded synthetic inputs -- TEST SIDE.

TEST INFRASTRUCTURE ONLY (same rules as oracle.py).  A restatement of the
product's config table (paper_1904_12380_b200/configs.py) whose bytes come
from the oracle's own C generators (sk_oracle.c), so the checker and the
``bench.py --impl reference`` arm never load the product library.
tests/test_oracle_golden.py pins this table to configs.py and the generated
bytes to the input SHA-256 recorded in tests/golden/golden.json.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

import oracle


@dataclass(frozen=True)
class Spec:
    name: str
    rows: int
    cols: int
    dist: str
    seed: int
    sigma: float = 1.0
    low: float = 0.0
    high: float = 1.0
    plant_count: int = 0
    plant_value: float = 0.0

    def describe(self) -> str:
        d = (f"N(0,{self.sigma:g}^2)" if self.dist == "normal"
             else f"U({self.low:g},{self.high:g})")
        s = f"{self.name} [{self.rows},{self.cols}] {d} seed {self.seed}"
        if self.plant_count:
            s += f", {self.plant_count} seeded positions = {self.plant_value:g}"
        return s


CONFIGS = {
    "c1": Spec("c1", 4096, 50, "normal", 0, sigma=4.0),
    "c2": Spec("c2", 65536, 128, "uniform", 1, low=-10.0, high=10.0),
    "c3": Spec("c3", 8192, 1000, "normal", 2, sigma=3.0, plant_count=81920, plant_value=-100.0),
    "c4": Spec("c4", 512, 262144, "normal", 3, sigma=5.0),
    "c5a": Spec("c5a", 2097152, 256, "normal", 4, sigma=1.0),
    "c5b": Spec("c5b", 1024, 1048576, "normal", 5, sigma=2.0),
}


def generate(name: str, row_start: int = 0, row_count: int | None = None,
             out: np.ndarray | None = None, nthreads: int = 0) -> np.ndarray:
    """Rows [row_start, row_start + row_count) of config `name` (float32)."""
    sp = CONFIGS[name]
    if row_count is None:
        row_count = sp.rows - row_start
    if row_start < 0 or row_count < 0 or row_start + row_count > sp.rows:
        raise ValueError("row range outside the config")
    if sp.plant_count and (row_start, row_count) != (0, sp.rows):
        raise ValueError(f"{name}: planted positions need the whole matrix")
    if out is None:
        out = np.empty((row_count, sp.cols), dtype=np.float32)
    flat = out.reshape(-1)
    L = oracle.lib()
    start = row_start * sp.cols
    if sp.dist == "normal":
        L.sko_fill_normal_f32(flat.ctypes.data, flat.size, sp.seed, sp.sigma, start, nthreads)
    else:
        L.sko_fill_uniform_f32(flat.ctypes.data, flat.size, sp.seed, sp.low, sp.high, start,
                               nthreads)
    if sp.plant_count:
        if L.sko_plant_f32(flat.ctypes.data, flat.size, sp.plant_count, sp.seed,
                           sp.plant_value) != 0:
            raise ValueError("plant failed")
    return out.reshape(row_count, sp.cols)


def sha256(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8).reshape(-1).data).hexdigest()
