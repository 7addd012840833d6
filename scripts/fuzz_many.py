#!/usr/bin/env python
"""Many seeds of tests/test_gpu_fuzz.py (one-off, not in the suite): 100 x 12 random cases."""
import sys, traceback
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import oracle
from tests import test_gpu_fuzz as f
fails = 0
for seed in range(100, 200):
    try:
        f.test_random_shapes_against_oracle(seed, oracle)
    except AssertionError as e:
        fails += 1
        print("FAIL seed", seed, str(e)[:600])
print("done fails", fails)
