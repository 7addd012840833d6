"""GPU checks of the round-1 advisor findings:

* K3g slot tags: the 23-bit launch epoch never wraps -- exchange blocks are
  zeroed every `gres_epoch_reset` launches (by the kernel for single-process
  blocks, CUDA-graph replays included; by sk_xchg_reset between barriers for
  cross-GPU blocks, which refuse to launch past the period);
* the torch ops record non-finite rows in the flag check_device_flag() reads;
* FusedColumnShard validates its tensors;
* the K1 / K1m thread-count knobs are rounded to whole warps / rows;
* the 1-D component ops return the reference's scan results for NaN / inf
  rows instead of raising.
"""

import numpy as np
import pytest
import torch

import paper_1904_12380_b200 as sk
from paper_1904_12380_b200 import _native, components, configs, sharding
from tests import gpu_util as gu

pytestmark = pytest.mark.gpu


def _bits(t):
    return t.contiguous().view(torch.int32).cpu().numpy()


@pytest.fixture
def period():
    def set_(n):
        _native.set_tuning("gres_epoch_reset", n)

    yield set_
    _native.set_tuning("gres_epoch_reset", 0)


def test_library_block_epoch_reset_keeps_bits(period):
    """Many K3g launches of different shapes on one stream with the block
    zeroed by the kernel every 1, 2, 3 launches: every result equals the
    result with the default period."""
    shapes = [(64, 262144), (40, 262144), (128, 131072), (300, 32768)]
    xs = [torch.from_numpy(configs.generate("c4", 0, r)[:, :c].copy()).cuda() for r, c in shapes]
    for r, c in shapes:
        assert gu.plan(r, c).startswith("k3_gres"), gu.plan(r, c)
    want = [sk.softmax(x, sk.KernelVariant.REFERENCE_CLIPPED) for x in xs]
    for n in (1, 2, 3):
        period(n)
        for it in range(3 * len(shapes) + 1):
            i = (it * 3) % len(shapes)  # interleave the shapes
            y = sk.softmax(xs[i], sk.KernelVariant.REFERENCE_CLIPPED)
            assert np.array_equal(_bits(y), _bits(want[i])), (n, it)


def test_library_block_epoch_reset_under_graph_replay(period):
    """The reset is device-driven, so graph replays (no host call per launch)
    cross reset boundaries correctly."""
    period(2)
    x = torch.from_numpy(configs.generate("c4", 0, 64)).cuda()
    ref = sk.softmax(x, sk.KernelVariant.REFERENCE_CLIPPED)
    out = torch.empty_like(x)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        sk.softmax_into(x, out, sk.KernelVariant.REFERENCE_CLIPPED, check_finite=False)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(3):
                sk.softmax_into(x, out, sk.KernelVariant.REFERENCE_CLIPPED, check_finite=False)
    for _ in range(7):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(_bits(out), _bits(ref))


def test_emulated_and_world_one_column_shard_resets(period, oracle):
    period(2)
    x = configs.generate("c4", 0, 6)[:, :160_000].copy()
    xd = torch.from_numpy(x).cuda()
    ref = oracle.softmax_ref(x, True, nthreads=0)
    for _ in range(5):
        y = sharding.emulate_column_shards(xd, sk.KernelVariant.REFERENCE_CLIPPED, 4)
        assert oracle.parity(y.cpu().numpy(), ref)["ok"]
    with sharding.FusedColumnShard() as fc:
        first = fc(xd, sk.KernelVariant.REFERENCE_CLIPPED)
        for _ in range(5):
            assert torch.equal(fc(xd, sk.KernelVariant.REFERENCE_CLIPPED), first)


def test_cross_gpu_block_refuses_past_the_period_until_reset(period):
    """A block with peers in other processes cannot be reset by the kernel:
    past the period the launch is refused until sk_xchg_reset."""
    from paper_1904_12380_b200.kernels import _bad_flag

    nat = sharding.NativeExchange()
    own, ghost = nat.alloc(0), nat.alloc(0)
    x = torch.from_numpy(configs.generate("c4", 0, 2)).cuda()
    y = torch.empty_like(x)
    flag = _bad_flag(torch, x.device)
    period(1)
    _native.set_tuning("gres_timeout_spins", 1 << 12)
    try:
        nat.launch(x, y, 0, 0, 2, [own, ghost], flag)  # the ghost never arrives: aborts
        torch.cuda.synchronize()
        flag.fill_(-1)
        with pytest.raises(sk.ArgumentError, match="sk_xchg_reset"):
            nat.launch(x, y, 0, 0, 2, [own, ghost], flag)
        nat.reset(own)
        nat.launch(x, y, 0, 0, 2, [own, ghost], flag)  # accepted again
        torch.cuda.synchronize()
        flag.fill_(-1)
    finally:
        _native.set_tuning("gres_timeout_spins", 0)
        nat.free(own)
        nat.free(ghost)


def test_torch_op_nonfinite_reaches_check_device_flag():
    from paper_1904_12380_b200 import torch_ops
    from paper_1904_12380_b200.kernels import check_device_flag

    ops = torch_ops.load()
    check_device_flag()  # clean start
    x = torch.from_numpy(configs.generate("c2", 0, 64)).cuda()
    x[17, 3] = float("nan")
    x[40, 0] = float("inf")
    ops.softmax_fwd(x, True)  # asynchronous: no raise here
    with pytest.raises(sk.NumericDomainError, match="row 17"):
        check_device_flag()
    check_device_flag()  # cleared
    m = ops.row_max(x)       # the stats kernels record into the same flag
    torch.cuda.synchronize()
    assert m.shape == (64,)
    with pytest.raises(sk.NumericDomainError, match="row 17"):
        check_device_flag()
    y = ops.softmax_fwd(x[:16].contiguous(), True)
    check_device_flag()  # finite rows: nothing recorded
    assert torch.isfinite(y).all()


def test_fused_column_shard_rejects_bad_tensors():
    x = torch.from_numpy(configs.generate("c4", 0, 4)).cuda()
    with sharding.FusedColumnShard() as fc:
        with pytest.raises(sk.ArgumentError, match="unit column stride"):
            fc(x[:, ::2], sk.KernelVariant.REFERENCE_CLIPPED)
        with pytest.raises(sk.ArgumentError, match="out must be"):
            fc(x, sk.KernelVariant.REFERENCE_CLIPPED, out=torch.empty(4, 10, device="cuda"))
        with pytest.raises(sk.ArgumentError, match="float32"):
            fc(x, sk.KernelVariant.REFERENCE_CLIPPED, out=torch.empty_like(x, dtype=torch.float64))
        with pytest.raises(sk.ArgumentError, match="unit column stride"):
            out = torch.empty(x.shape[1], x.shape[0], device="cuda").t()
            fc(x, sk.KernelVariant.REFERENCE_CLIPPED, out=out)
        y = fc(x, sk.KernelVariant.REFERENCE_CLIPPED)
        assert torch.isfinite(y).all()


@pytest.mark.parametrize("key,value,shape", [("k1_threads", 96, (3000, 128)),
                                             ("k1_threads", 200, (3000, 1000)),
                                             ("k1m_threads", 96, (700, 4096)),
                                             ("k1m_threads", 200, (700, 1501))])
def test_thread_knobs_round_to_whole_warps_and_rows(key, value, shape, oracle):
    x = configs.generate("c4", 0, shape[0] * shape[1] // 262144 + 1).reshape(-1)
    x = np.ascontiguousarray(x[:shape[0] * shape[1]].reshape(shape))
    ref = oracle.softmax_ref(x, True, nthreads=0)
    _native.set_tuning(key, value)
    try:
        y, bad = gu.softmax_abi(x)
        p = gu.plan(*shape)
    finally:
        _native.set_tuning(key, 128 if key == "k1_threads" else 0)
    assert bad == gu.NO_BAD
    threads = int(p.split("threads=")[1].split()[0])
    assert threads % 32 == 0, p
    assert oracle.parity(y, ref)["ok"], p


ROWS = [
    [np.nan, 1.0, 2.0], [1.0, np.nan, 2.0], [1.0, np.inf, 2.0], [-np.inf, -np.inf],
    [1.0, -np.inf, 3.0], [np.inf, np.nan], [-np.inf, 0.5], [np.inf, np.inf, -1.0],
]


@pytest.mark.parametrize("row", ROWS)
def test_component_ops_nonfinite_rows_follow_the_reference(row, oracle):
    """kernels.py:229-231 / 272-276: a strict '>' scan from a[0] and the f64
    sum of exp(row - max) -- defined results, no error, for NaN / inf rows."""
    a = np.array(row, np.float32)
    m_ref = oracle.row_max_scalar(a)
    st_ref = oracle.row_stats(a)
    m = components.row_max_scalar(a)
    st = components.row_stats(a)
    for got, want in ((m, m_ref), (st.max, st_ref[0])):
        assert (np.isnan(got) and np.isnan(want)) or got == want, (row, got, want)
    s, s_ref = np.float32(st.sum), np.float32(st_ref[1])
    if np.isfinite(s_ref):
        assert abs(float(s) - float(s_ref)) <= 2 * np.spacing(s_ref), (row, s, s_ref)
    else:
        assert (np.isnan(s) and np.isnan(s_ref)) or s == s_ref, (row, s, s_ref)
    # device tensors too
    md = components.row_max_scalar(torch.from_numpy(a).cuda())
    assert (bool(torch.isnan(md)) and np.isnan(m_ref)) or float(md) == float(m_ref)


def test_every_plan_kind_interleaved(oracle):
    """Jobs of every plan kind -- K1, K1m, K2 (k1m off), K3g over aligned and
    unaligned rows, the split path -- interleaved on one stream, twice: no
    launch inherits anything from the previous one (workspace, K3g exchange
    block, plan fields), each result against the oracle.  (A per-thread plan
    cache tried this round leaked a K3g plan's fields into a K2 launch; it
    measured no faster and was removed.)"""
    shapes = [(4096, 128), (64, 4096), (40, 6144), (64, 262144), (400, 50257), (3, 300000),
              (700, 1000), (33, 16384), (64, 65536), (1500, 50), (20, 8192)]
    xs = {s: configs.generate("c4", 0, -(-s[0] * s[1] // 262144)).reshape(-1)[:s[0] * s[1]]
          .reshape(s).copy() for s in shapes}
    refs = {s: oracle.softmax_ref(xs[s], True, nthreads=0) for s in shapes}
    _native.set_tuning("k1m", 0)  # 4096 / 6144 / 8192 columns take K2 (kPathSeg, k3 unset)
    try:
        kinds = set()
        for _ in range(2):
            for s in shapes:
                kinds.add(gu.plan(*s).split()[0])
                y, bad = gu.softmax_abi(xs[s])
                assert bad == gu.NO_BAD
                assert oracle.parity(y, refs[s])["ok"], (s, gu.plan(*s))
        assert {"k1", "k2_tma", "k3_gres", "k3_gres_unal", "k4_split"} <= kinds, kinds
    finally:
        _native.set_tuning("k1m", 1)
