"""Timing chaos for the barrier-heavy long-row kernel (K3g): with gres_diag
bit 6 every warp sleeps a pseudo-random 0-4 us at each hand-off point (stage
wait, named-barrier arrive / sync, slot publication, TMA refill, poll, output),
a different schedule per seed.  The pool's GPUs refuse compute-sanitizer's
racecheck / synccheck, so this is the stand-in: a dependency the barriers,
mbarriers or epoch-tagged slots fail to enforce shows up as changed bits, a
wrong answer or an exchange timeout under some schedule."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture
def tuning():
    from paper_1904_12380_b200 import _native

    yield _native
    _native.set_tuning("gres_diag", 0)
    _native.set_tuning("gres", 1)


def _chaos_runs(tuning, fn, seeds=(1, 2, 3, 4)):
    import torch

    tuning.set_tuning("gres_diag", 0)
    y0 = fn()
    torch.cuda.synchronize()
    for seed in seeds:
        tuning.set_tuning("gres_diag", 64 | ((seed * 7919) << 8))
        y = fn()
        torch.cuda.synchronize()
        assert torch.equal(y, y0), f"bits changed under schedule seed {seed}"
    tuning.set_tuning("gres_diag", 0)
    return y0


@pytest.mark.timeout(600)
@pytest.mark.parametrize("rows,cols,what", [
    (96, 262144, "c4-like: 14 CTAs per row, publisher polls (lag 1)"),
    (40, 1048576, "c5b-like: 74 CTAs per row, separate poller warp (lag 2)"),
    (300, 32768, "2 CTAs per row, 74 row groups"),
    (512, 50257, "unaligned rows: per-row slice geometry, head / tail floats"),
    (2048, 20000, "one CTA per row: the ring and its barriers without a group"),
])
def test_k3g_bits_do_not_depend_on_timing(tuning, oracle, rows, cols, what):
    import torch

    import paper_1904_12380_b200 as sk

    tuning.set_tuning("gres", 2)  # K3g even where a small job would take the latency path
    plan = tuning.describe_plan(rows, cols)
    assert plan.startswith("k3_gres"), plan
    rng = np.random.default_rng(rows * 31 + cols)
    x_host = (rng.standard_normal((rows, cols), dtype=np.float32) * 5).astype(np.float32)
    x_host[rng.integers(0, rows, 64), rng.integers(0, cols, 64)] = -100.0  # clip fires
    x = torch.from_numpy(x_host).cuda()
    y0 = _chaos_runs(tuning, lambda: sk.softmax(x, sk.KernelVariant.REFERENCE_CLIPPED))
    chk = slice(0, min(rows, 24))
    d = oracle.parity(y0[chk].cpu().numpy(), oracle.softmax_ref(x_host[chk], True))
    assert d["ok"], (what, d)


@pytest.mark.timeout(600)
def test_fused_column_shard_bits_do_not_depend_on_timing(tuning, oracle):
    """Four ranks' shards in one cooperative launch: every CTA publishes into
    every rank's exchange block and polls its own, under shaken schedules."""
    import torch

    import paper_1904_12380_b200 as sk
    from paper_1904_12380_b200 import sharding

    rng = np.random.default_rng(77)
    x_host = (rng.standard_normal((48, 4 * 65536), dtype=np.float32) * 3).astype(np.float32)
    x = torch.from_numpy(x_host).cuda()
    y0 = _chaos_runs(tuning, lambda: sharding.emulate_column_shards(
        x, sk.KernelVariant.REFERENCE_CLIPPED, 4), seeds=(5, 6, 7))
    d = oracle.parity(y0[:16].cpu().numpy(), oracle.softmax_ref(x_host[:16], True))
    assert d["ok"], d


@pytest.mark.timeout(600)
def test_k3c_cluster_rows_bits_do_not_depend_on_timing(tuning, oracle):
    """The cluster-resident fallback (K3c: DSMEM st.async pushes completing
    peers' mbarriers, a TMA ring per CTA) under the same shaken schedules."""
    import torch

    import paper_1904_12380_b200 as sk

    rows, cols = 160, 131072
    tuning.set_tuning("gres", 0)
    tuning.set_tuning("k3_impl", 5)
    try:
        plan = tuning.describe_plan(rows, cols)
        assert plan.startswith("k3_cluster"), plan
        rng = np.random.default_rng(5)
        x_host = (rng.standard_normal((rows, cols), dtype=np.float32) * 5).astype(np.float32)
        x = torch.from_numpy(x_host).cuda()
        y0 = _chaos_runs(tuning, lambda: sk.softmax(x, sk.KernelVariant.REFERENCE_CLIPPED))
        d = oracle.parity(y0[:16].cpu().numpy(), oracle.softmax_ref(x_host[:16], True))
        assert d["ok"], d
    finally:
        tuning.set_tuning("k3_impl", 3)


@pytest.mark.timeout(600)
def test_fused_column_shard_with_system_scope_slot_accesses(tuning, oracle):
    """The cross-GPU launch publishes and polls its slots with st / ld.relaxed.sys
    (peer memory over NVLink).  One GPU cannot run two ranks' kernels that wait
    on each other, so the emulated 4-rank launch is switched to the same
    system-scope accesses (colshard_sys): same bits as the .gpu-scope run, also
    under shaken schedules."""
    import torch

    import paper_1904_12380_b200 as sk
    from paper_1904_12380_b200 import sharding

    rng = np.random.default_rng(91)
    x_host = (rng.standard_normal((40, 4 * 50000), dtype=np.float32) * 3).astype(np.float32)
    x = torch.from_numpy(x_host).cuda()
    fn = lambda: sharding.emulate_column_shards(x, sk.KernelVariant.REFERENCE_CLIPPED, 4)  # noqa: E731
    y_gpu = fn()
    tuning.set_tuning("colshard_sys", 1)
    try:
        y_sys = _chaos_runs(tuning, fn, seeds=(11, 12, 13))
    finally:
        tuning.set_tuning("colshard_sys", 0)
    assert torch.equal(y_sys, y_gpu)
    d = oracle.parity(y_sys[:16].cpu().numpy(), oracle.softmax_ref(x_host[:16], True))
    assert d["ok"], d
