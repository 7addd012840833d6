"""GPU tests of the sharding layer on one B200.

Only one GPU is available per run, so n-way column sharding is emulated on
one device: each shard runs the real native kernels (sk_row_stats_f32 /
sk_rescale_sumexp / sk_normalize_f32); the all-reduce is replaced by the
equivalent torch max / sum over the shard statistics.  The real NCCL path
runs at world size 1.  (Multi-rank collectives are covered on CPU by
tests/test_sharding_gloo.py.)
"""

import os
import socket

import numpy as np
import pytest
import torch

import paper_1904_12380_b200 as sk
from paper_1904_12380_b200 import configs, sharding

pytestmark = pytest.mark.gpu


def _emulated_column_softmax(x, n, variant):
    ops = sharding.cuda_column_ops()
    mode = sk.variant_mode(variant)
    cols = x.shape[1]
    spans = [sharding.shard_range(cols, n, r) for r in range(n)]
    shards = [x[:, a:a + w].contiguous() for a, w in spans]
    stats = [ops.local_stats(s, mode) for s in shards]
    M = torch.stack([m for m, _ in stats]).max(dim=0).values          # all_reduce(MAX)
    S = sum(ops.rescale(m, M, s.clone()) for m, s in stats)           # all_reduce(SUM)
    return torch.cat([ops.normalize(s, M, S, mode) for s in shards], dim=1)


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_column_shards_emulated_c5b_rows(n, oracle):
    spec = configs.get("c5b")
    x = configs.generate(spec, 0, 6)
    xd = torch.from_numpy(x).cuda()
    y = _emulated_column_softmax(xd, n, sk.KernelVariant.REFERENCE_CLIPPED).cpu().numpy()
    d = oracle.parity(y, oracle.softmax_ref(x, True, nthreads=0))
    assert d["ok"], (n, d)


@pytest.mark.parametrize("n", [2, 3, 8])
def test_column_shards_emulated_clip_and_ragged(n, oracle):
    x = np.ascontiguousarray(configs.generate("c3")[:200, :997])
    xd = torch.from_numpy(x).cuda()
    for v in (sk.KernelVariant.REFERENCE_CLIPPED, sk.KernelVariant.REFERENCE_INFERENCE):
        y = _emulated_column_softmax(xd, n, v).cpu().numpy()
        ref = oracle.softmax_ref(x, v is sk.KernelVariant.REFERENCE_CLIPPED)
        assert oracle.parity(y, ref)["ok"], (n, v)


def test_nccl_world_size_one(oracle):
    import torch.distributed as dist

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        x = configs.generate("c5b", 0, 4)
        xd = torch.from_numpy(x).cuda()
        y = sharding.column_sharded_softmax(xd, sk.KernelVariant.REFERENCE_CLIPPED)
        assert oracle.parity(y.cpu().numpy(), oracle.softmax_ref(x, True, nthreads=0))["ok"]
        yr = sharding.row_sharded_softmax(xd, sk.KernelVariant.REFERENCE_CLIPPED)
        assert oracle.parity(yr.cpu().numpy(), oracle.softmax_ref(x, True, nthreads=0))["ok"]
    finally:
        dist.destroy_process_group()


def test_row_stats_device_matches_full_softmax(oracle):
    x = configs.generate("c4", 0, 3)
    st = sk.row_stats_device(torch.from_numpy(x).cuda())
    m = x.max(axis=1)
    assert np.array_equal(st.max.cpu().numpy(), m)
    s = np.exp(np.maximum(x - m[:, None], -64).astype(np.float64)).sum(axis=1)
    np.testing.assert_allclose(st.sum.cpu().numpy(), s, rtol=1e-6)


# ------------------------------------------------------- fused column shard
def _plan_ok(rows, cols, world):
    from paper_1904_12380_b200 import _native

    d = _native.describe_colshard_plan(rows, cols // world, world, emulate=True)
    assert d.startswith("k3_gres_colshard world=%d nvr=%d " % (world, world)), d
    return d


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_fused_column_shards_emulated_c5b_rows(world, oracle):
    """All `world` ranks of the fused column shard as one cooperative kernel:
    c5b rows (1M columns) match the oracle of the full rows."""
    spec = configs.get("c5b")
    x = configs.generate(spec, 0, 6)
    _plan_ok(6, spec.cols, world)
    y = sharding.emulate_column_shards(torch.from_numpy(x).cuda(),
                                       sk.KernelVariant.REFERENCE_CLIPPED, world)
    d = oracle.parity(y.cpu().numpy(), oracle.softmax_ref(x, True, nthreads=0))
    assert d["ok"], (world, d)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_fused_column_shards_modes_clip_ragged(world, oracle):
    """Every mode; the clip fires in one shard only; a large negative row; a
    shard width whose last CTA slice is ragged; more row groups than rows."""
    C = 24_000 * world
    x = configs.generate("c4", 0, 13)[:, :C].copy()
    x[3, 777] = -500.0
    x[5, :] -= 400.0
    x[7, C - 3] = 90.0  # the row max lives in the last shard
    xd = torch.from_numpy(x).cuda()
    for v in (sk.KernelVariant.REFERENCE_CLIPPED, sk.KernelVariant.REFERENCE_INFERENCE,
              sk.KernelVariant.FULL_VECTORIZED_APPROX_EXP):
        y = sharding.emulate_column_shards(xd, v, world).cpu().numpy()
        ref = oracle.softmax_ref(x, v is sk.KernelVariant.REFERENCE_CLIPPED)
        d = oracle.parity(y, ref, approx=v is sk.KernelVariant.FULL_VECTORIZED_APPROX_EXP)
        assert d["ok"], (world, v, d)


def test_fused_column_shards_full_c5b():
    """Full c5b (1024 x 1048576) over 8 emulated ranks: every row sums to 1 and
    the result equals the single-GPU softmax within the fp32 tolerance."""
    spec = configs.get("c5b")
    xd = torch.from_numpy(configs.generate(spec)).cuda()
    y8 = sharding.emulate_column_shards(xd, sk.KernelVariant.REFERENCE_CLIPPED, 8)
    y1 = sk.softmax(xd, sk.KernelVariant.REFERENCE_CLIPPED)
    torch.cuda.synchronize()
    rs = torch.stack([y8[i].double().sum() for i in range(spec.rows)])
    assert float((rs - 1).abs().max()) <= 1e-5
    assert float((y8 - y1).abs().max()) <= 1e-6
    assert float(((y8 - y1).abs() / y1).max()) <= 1e-5


def test_fused_column_shard_world_one_api(oracle):
    """FusedColumnShard through its public API at world size 1 (IPC handle of
    the exchange block taken, no peers opened)."""
    x = configs.generate("c4", 0, 9)
    with sharding.FusedColumnShard() as fc:
        assert fc.world == 1 and fc.blocks == [fc.block]
        y = fc(torch.from_numpy(x).cuda(), sk.KernelVariant.REFERENCE_CLIPPED)
        y2 = fc(torch.from_numpy(x).cuda(), sk.KernelVariant.REFERENCE_CLIPPED)
    assert torch.equal(y, y2)
    assert oracle.parity(y.cpu().numpy(), oracle.softmax_ref(x, True, nthreads=0))["ok"]


def test_fused_column_shard_nonfinite_row():
    x = configs.generate("c4", 0, 12)[:, :160_000].copy()
    x[9, 100_001] = np.nan   # shard 2 of 4
    x[11, 5] = np.inf        # shard 0
    with pytest.raises(sk.NumericDomainError, match="row 9"):
        sharding.emulate_column_shards(torch.from_numpy(x).cuda(),
                                       sk.KernelVariant.REFERENCE_CLIPPED, 4)
    y = sharding.emulate_column_shards(torch.ones(3, 160_000, device="cuda"),
                                       sk.KernelVariant.REFERENCE_CLIPPED, 4)
    assert torch.allclose(y, torch.full_like(y, 1 / 160_000))


def test_fused_column_shard_missing_peer_times_out(oracle):
    """A rank whose peer never launches must not hang the GPU: the exchange
    aborts after its spin budget, the call raises, and the next call is clean."""
    from paper_1904_12380_b200 import _native
    from paper_1904_12380_b200.kernels import _bad_flag, _raise_if_aborted

    nat = sharding.NativeExchange()
    own, ghost = nat.alloc(0), nat.alloc(0)
    x = torch.from_numpy(configs.generate("c4", 0, 4)).cuda()
    y = torch.empty_like(x)
    flag = _bad_flag(torch, x.device)
    _native.set_tuning("gres_timeout_spins", 1 << 14)
    try:
        nat.launch(x, y, 0, 0, 2, [own, ghost], flag)  # rank 1 never runs
        with pytest.raises(sk.SoftmaxKitError, match="timed out"):
            _raise_if_aborted(flag, int(flag.item()))
        with sharding.FusedColumnShard() as fc:  # a fresh, healthy exchange
            y1 = fc(x, sk.KernelVariant.REFERENCE_CLIPPED)
        assert oracle.parity(y1.cpu().numpy(), oracle.softmax_ref(x.cpu().numpy(), True))["ok"]
        nat.launch(x, y, 0, 0, 1, [own], flag)  # the aborted block recovers too
        assert int(flag.item()) == -1
        assert oracle.parity(y.cpu().numpy(), oracle.softmax_ref(x.cpu().numpy(), True))["ok"]
    finally:
        _native.set_tuning("gres_timeout_spins", 0)
        nat.free(own)
        nat.free(ghost)


def test_fused_column_shards_graph_replay(oracle):
    """The launch epoch lives on the device, so CUDA-graph replays of the fused
    kernel stay correct (stale slots of the previous replay are never taken)."""
    xs = [configs.generate("c4", 0, 8) + np.float32(i) * 0.37 for i in range(2)]
    xd = torch.from_numpy(xs[0]).cuda()
    out = torch.empty_like(xd)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        sharding.emulate_column_shards(xd, sk.KernelVariant.REFERENCE_CLIPPED, 4, out=out,
                                       check_finite=False)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            sharding.emulate_column_shards(xd, sk.KernelVariant.REFERENCE_CLIPPED, 4, out=out,
                                           check_finite=False)
    for it in range(4):
        xd.copy_(torch.from_numpy(xs[it % 2]))
        g.replay()
        torch.cuda.synchronize()
        ref = oracle.softmax_ref(xs[it % 2], True, nthreads=0)
        assert oracle.parity(out.cpu().numpy(), ref)["ok"], it
