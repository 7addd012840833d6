#!/usr/bin/env python
"""Many seeds of tests/test_gpu_fuzz.py::test_random_short_rows_against_oracle
(one-off, not in the suite): K1 short / medium rows at random lengths, job
sizes, base offsets, pitches and modes against the oracle."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import oracle  # noqa: E402
from tests import test_gpu_fuzz as f  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
fails = 0
for seed in range(100, 100 + n):
    try:
        f.test_random_short_rows_against_oracle(seed, oracle)
    except AssertionError as e:
        fails += 1
        print("FAIL seed", seed, str(e)[:600], flush=True)
print("done seeds", n, "fails", fails)
