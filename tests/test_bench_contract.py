"""bench.py contract checks that run on CPU: the reference arm (CPU by
definition) prints one JSON line with the driver's keys."""

import json
import subprocess
import sys

from tests.conftest import ROOT


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                        "--steps", "3", "--warmup", "1"], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["workload"].startswith("c2")


def _torchrun(nproc, *args, env=None, timeout=600):
    import os

    e = dict(os.environ, **(env or {}))
    return subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                           f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1",
                           "--master-port", str(29500 + os.getpid() % 1000),
                           str(ROOT / "bench.py"), "--gpus", str(nproc), *args],
                          capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=e)


def test_reference_arm_under_torchrun_rank0_only():
    """The driver launches the reference arm with torchrun for N>1: rank 0
    alone times the CPU path and prints one line; other ranks exit 0."""
    r = _torchrun(2, "--impl", "reference", "--steps", "2", "--warmup", "1")
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
