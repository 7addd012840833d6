"""Shared test setup.

Markers: ``gpu`` tests need a B200 (run via gpurun); everything else runs on
CPU.  The oracle (oracle/) is test infrastructure and is imported only here
and in tests.
"""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires an NVIDIA B200 (sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN / "golden.npz")


@pytest.fixture(scope="session")
def golden_components():
    return np.load(GOLDEN / "golden_components.npz")


@pytest.fixture(scope="session")
def golden_meta():
    import json

    return json.loads((GOLDEN / "golden.json").read_text())


@pytest.fixture(scope="session")
def oracle():
    import oracle as o

    o.lib()
    return o


@pytest.fixture(scope="session")
def native():
    from paper_1904_12380_b200 import _native

    _native.lib()
    return _native
