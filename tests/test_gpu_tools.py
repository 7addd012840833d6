"""GPU tests of the phase pipeline, profiler, bound probe and CLI."""

import numpy as np
import pytest
import torch

import paper_1904_12380_b200 as sk
from paper_1904_12380_b200 import bench_cli, bound_probe, configs, phases, profiler

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("C", [1, 50, 1000, 4097, 70000])
def test_phase_pipeline_matches_fused(C, oracle):
    x = configs.generate("c4", 0, 7)[:, :C].copy()
    xd = torch.from_numpy(x).cuda()
    for v in (sk.KernelVariant.REFERENCE_CLIPPED, sk.KernelVariant.REFERENCE_INFERENCE):
        pipe = phases.variant_pipeline(v, *x.shape)
        buf = torch.empty_like(xd)
        pipe.maxsub(xd, buf)
        pipe.exp(buf)
        pipe.sumscale(buf)
        ref = oracle.softmax_ref(x, v is sk.KernelVariant.REFERENCE_CLIPPED)
        assert oracle.parity(buf.cpu().numpy(), ref)["ok"], (C, v)


def test_profiler_and_probe_on_gpu():
    m = sk.Matrix2D.from_array(configs.generate("c3"))
    t = profiler.time_phases(m, sk.KernelVariant.REFERENCE_CLIPPED, reps=20, warmup=3)
    assert all(x.phase_sum <= x.whole for x in t)
    w = profiler.time_whole(m, sk.KernelVariant.REFERENCE_CLIPPED, reps=20, warmup=3)
    assert min(w) > 0
    r = bound_probe.probe(m, sk.KernelVariant.REFERENCE_CLIPPED, reps=20, warmup=3)
    print("c3 probe", r)
    # the fused kernel moves the copy's bytes at the copy's speed: memory bound
    assert r.verdict is bound_probe.Verdict.MEMORY_BOUND_LIKELY
    s = bound_probe.probe_self_copy(m, reps=20, warmup=3)
    assert s.verdict is bound_probe.Verdict.MEMORY_BOUND_LIKELY


def test_cli_verify_and_bench(capsys):
    assert bench_cli.main(["verify", "--reps", "5"]) == 0
    out = capsys.readouterr().out
    assert "verify: OK" in out
    assert bench_cli.main(["bench", "--reps", "10", "--format", "csv",
                           "--batch-size", "32", "--batch-size", "128"]) == 0
    rows = capsys.readouterr().out.strip().splitlines()
    assert rows[0].startswith("variant,batch,cols,median_ticks")
    assert len(rows) == 1 + 2 * (len(sk.LADDER) + 1)
    assert bench_cli.main(["probe", "--reps", "5", "--batch-size", "128"]) == 0
    assert "CopyBaseline" in capsys.readouterr().out
    assert bench_cli.main(["profile", "--reps", "5", "--batch-size", "8",
                           "--variant", "ReferenceClipped"]) == 0
    assert "Profiling Report" in capsys.readouterr().out


def test_bench_colshard_mode():
    """bench.py --colshard (the fused column shard's benchmark) at world size 1:
    one JSON line with the contract's keys, parity against the oracle."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--config", "c4", "--colshard",
                        "--steps", "12", "--warmup", "3", "--e2e-steps", "1"],
                       capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    for k in ("metric", "value", "unit", "n_gpus", "ms_per_step", "roofline", "e2e",
              "gpu_launches", "clocks", "config"):
        assert k in line, k
    assert line["config"]["plan"].startswith("k3_gres_colshard world=1")
    assert line["parity"]["ok"], line["parity"]
    assert line["value"] > 1000


def test_bench_row_shard_under_torchrun():
    """bench.py's N>1 row-shard path (torchrun, barrier, max-over-ranks) at
    world size 2 on one GPU: SK_BENCH_SHARE_DEVICE puts both ranks on cuda:0
    over gloo (row shards never wait on each other; the numbers mean nothing,
    the code path is what is checked)."""
    import json

    from tests.test_bench_contract import _torchrun

    r = _torchrun(2, "--config", "c2", "--extra", "", "--steps", "64", "--warmup", "3",
                  "--e2e-steps", "1", "--no-cpu-baseline", env={"SK_BENCH_SHARE_DEVICE": "1"})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["rows"] == 65536
    assert d["setup"]["rows_per_gpu"] == 32768 and d["scaling"] == "strong"
    assert d["parity"]["ok"] and d["parity"]["rows_checked"] == 65536
    assert d["e2e"]["bitwise_equal_device_path"] and d["e2e"]["pinned"]["bitwise_equal_device_path"]
    assert d["gpu_launches"] == 64 and d["value"] > 0
