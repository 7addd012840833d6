"""GPU parity: the CUDA path (through the C ABI) against the reference.

Gate (BASELINE.json north_star): max |d| <= 1e-6, max |d|/ref <=
1e-5, max |rowsum - 1| <= 1e-5 against ReferenceClipped on identical inputs;
1e-5 relative for the approximate-exp rung (reference bench.py:52).  Small
cases compare straight against outputs of the reference itself
(tests/golden); full configs against the C oracle, which is pinned
bit-exact to the reference (test_oracle_golden.py).
"""

import numpy as np
import pytest

import paper_1904_12380_b200 as sk
from paper_1904_12380_b200 import _native, configs
from tests import gpu_util as gu

pytestmark = pytest.mark.gpu

MODES = {"clipped": 0, "inference": 1, "approx": 2}


def assert_parity(oracle, y, ref, approx=False, what=""):
    d = oracle.parity(y, ref, approx=approx)
    assert d["ok"], (what, d)
    return d


@pytest.fixture(autouse=True)
def _reset_tuning():
    yield
    for k, v in (("path", -1), ("k1_lpr", 0), ("grid_mult", 0),
                 ("skip_max_shift", 0), ("k3_impl", 3), ("cluster_k3", 1),
                 ("gres", 1), ("gres_p", 0), ("gres_st", 0), ("gres_lag", 0), ("gres_split", -1), ("cluster_onex", 0), ("k1m", 1),
                 ("k1m_wpr", 0), ("k1m_nv", 0), ("k1_nv", 0), ("k1_u", 0), ("k1_pf", -1),
                 ("vec2_max", 128)):
        _native.set_tuning(k, v)


# ---------------------------------------------------------------- golden sweep
def test_sweep_against_reference_outputs(golden, golden_meta, oracle):
    for C in golden_meta["sweep"]:
        x = golden[f"sweep/{C}/x"]
        for rung, mode in MODES.items():
            y, bad = gu.softmax_abi(x, mode)
            assert bad == gu.NO_BAD
            assert_parity(oracle, y, golden[f"sweep/{C}/{rung}"], approx=(mode == 2),
                          what=(C, rung, gu.plan(*x.shape)))


def test_spec_known_answers(golden, oracle):
    for case in ("spec_123", "spec_zeros", "spec_single", "spec_big", "spec_clip"):
        x = golden[f"{case}/x"]
        for rung in ("clipped", "inference"):
            y, _ = gu.softmax_abi(x, MODES[rung])
            assert_parity(oracle, y, golden[f"{case}/{rung}"], what=(case, rung))
    y, _ = gu.softmax_abi(np.array([[3.0]], np.float32))
    assert y[0, 0] == 1.0
    y, _ = gu.softmax_abi(np.zeros((1, 4), np.float32))
    assert np.all(y == 0.25)
    x = np.array([[0.0, -100.0]], np.float32)
    assert gu.softmax_abi(x, 0)[0][0, 1] > 0
    assert gu.softmax_abi(x, 1)[0][0, 1] == 0


def test_config_rows_against_reference(golden, oracle):
    for name in ("c1", "c3"):
        y, _ = gu.softmax_abi(golden[f"{name}/x"], 0)
        assert_parity(oracle, y, golden[f"{name}/clipped"], what=name)


# ---------------------------------------------------------------- full configs
@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_config_full_parity(name, oracle):
    x = configs.generate(name)
    ref = oracle.softmax_ref(x, True, nthreads=0)
    y, bad = gu.softmax_abi(x, 0)
    assert bad == gu.NO_BAD
    d = assert_parity(oracle, y, ref, what=(name, gu.plan(*x.shape)))
    print(name, gu.plan(*x.shape), d)


@pytest.mark.parametrize("name", ["c4", "c5a", "c5b"])
def test_config_full_every_element(name, oracle):
    """Full-size run through the public API: EVERY output element of the
    config against the oracle (bit-exact C restatement of ReferenceClipped),
    at the north-star gate, like the reference harness verifies every row
    (bench.py:160-185)."""
    t = gu.torch()
    spec = configs.get(name)
    x = configs.generate(spec)
    xd = t.from_numpy(x).cuda()
    yd = sk.softmax(xd, sk.KernelVariant.REFERENCE_CLIPPED)
    t.cuda.synchronize()
    del xd
    d = gu.parity_all_rows(oracle, yd, x)
    print(name, gu.plan(spec.rows, spec.cols), d)
    assert d["ok"], (name, d)
    assert d["rows_checked"] == spec.rows


@pytest.mark.parametrize("world", [2, 4, 8])
def test_c5b_column_shards_every_element(world, oracle):
    """c5b split by columns over `world` ranks, all ranks' fused kernels
    emulated as one cooperative launch on this GPU (the same publish / poll
    exchange code as the per-rank NVLink kernel): every element of the full
    [1024, 1048576] output against the oracle."""
    from paper_1904_12380_b200 import sharding

    t = gu.torch()
    spec = configs.get("c5b")
    x = configs.generate(spec)
    xd = t.from_numpy(x).cuda()
    yd = sharding.emulate_column_shards(xd, sk.KernelVariant.REFERENCE_CLIPPED, world)
    t.cuda.synchronize()
    del xd
    d = gu.parity_all_rows(oracle, yd, x)
    print("c5b colshard", world, d)
    assert d["ok"], (world, d)


# ---------------------------------------------------------------- edge shapes
EDGE_C = [1, 2, 3, 7, 49, 50, 51, 127, 128, 129, 1000, 1023, 1024, 1025, 4096, 4097, 8192,
          8193, 12289, 65536, 65537, 262144]


@pytest.mark.parametrize("C", EDGE_C)
def test_edge_shapes(C, oracle):
    rows = 37 if C <= 8193 else 5
    x = np.empty((rows, C), np.float32)
    from paper_1904_12380_b200 import tensor

    tensor.fill_normal_array(x, C, 6.0)
    if C > 5:
        x[1, C // 2] = -300.0  # clip fires
        x[2, :] -= 500.0       # large negative row (shift invariance)
    for mode in (0, 1):
        ref = oracle.softmax_ref(x, clip=(mode == 0))
        y, bad = gu.softmax_abi(x, mode)
        assert bad == gu.NO_BAD
        assert_parity(oracle, y, ref, what=(C, mode, gu.plan(rows, C)))


@pytest.mark.parametrize("C", [50, 128, 1000, 2048, 4097, 16384, 100000])
def test_unaligned_and_strided(C, oracle):
    rows = 9
    x = np.empty((rows, C), np.float32)
    from paper_1904_12380_b200 import tensor

    tensor.fill_uniform_array(x, 11, -30, 30)
    ref = oracle.softmax_ref(x)
    for xo, yo, ldx, ldy in ((1, 0, None, None), (0, 3, None, None), (0, 0, C + 4, C + 8),
                             (2, 1, C + 3, C + 5)):
        y, _ = gu.softmax_abi(x, 0, x_offset=xo, y_offset=yo, ldx=ldx, ldy=ldy)
        assert_parity(oracle, y, ref, what=(C, xo, yo, ldx, ldy))


@pytest.mark.parametrize("path", [0, 1, 2, 3])
def test_every_path_on_same_input(path, oracle):
    C = 1024 if path == 0 else 8192 if path == 3 else 20000
    x = configs.generate("c4", 0, 3)[:, :C].copy()
    ref = oracle.softmax_ref(x)
    _native.set_tuning("path", path)
    y, _ = gu.softmax_abi(x, 0)
    assert_parity(oracle, y, ref, what=path)


def test_k1_instantiations_all_agree(oracle):
    x = configs.generate("c2", 0, 999)
    ref = oracle.softmax_ref(x)
    shapes = ((4, 8, 4, 1), (4, 8, 4, 2), (4, 16, 2, 2), (4, 16, 4, 1), (4, 32, 1, 4),
              (4, 32, 4, 1), (8, 16, 1, 2), (8, 8, 2, 1), (8, 32, 1, 1))
    try:
        for vec, lpr, nv, u in shapes:
            _native.set_tuning("vec8", 1 if vec == 8 else 0)
            _native.set_tuning("k1_lpr", lpr)
            _native.set_tuning("k1_nv", nv)
            _native.set_tuning("k1_u", u)
            for pf in (0, 1) if (vec, lpr, nv, u) == (4, 8, 4, 1) else (0,):
                _native.set_tuning("k1_pf", pf)
                y, _ = gu.softmax_abi(x, 0)
                assert_parity(oracle, y, ref, what=(vec, lpr, nv, u, pf))
    finally:
        _native.set_tuning("vec8", 0)
        _native.set_tuning("k1_pf", -1)


@pytest.mark.parametrize("rows,C", [(8, 50257), (32, 151936), (3, 20000), (40, 262147)])
def test_split_fused_combine_keeps_bits(rows, C, oracle):
    """The split path with the row statistics merged inside the normalize pass
    (two launches) gives the three-launch path's bits, and both match the oracle."""
    from paper_1904_12380_b200 import tensor

    x = np.empty((rows, C), np.float32)
    tensor.fill_normal_array(x, C + rows, 5.0)
    x[1, 7] = -500.0
    ref = oracle.softmax_ref(x)
    outs = []
    try:
        _native.set_tuning("path", 2)
        for fuse in (0, 1, 2):
            _native.set_tuning("k4_fuse_combine", fuse)
            y, bad = gu.softmax_abi(x, 0)
            assert bad == gu.NO_BAD
            assert_parity(oracle, y, ref, what=(rows, C, fuse))
            outs.append(y)
    finally:
        _native.set_tuning("k4_fuse_combine", 1)
    assert all(np.array_equal(o.view(np.uint32), outs[0].view(np.uint32)) for o in outs[1:])


def test_k1_vec2_instantiations_all_agree(oracle):
    """Every 64-bit K1 instantiation (even rows on 8-B pitches) against the
    oracle, on row lengths it covers, plus the 32-bit plan of the same rows."""
    from paper_1904_12380_b200 import tensor

    shapes = {10: ((4, 2, 4, 0), (4, 2, 8, 0), (8, 1, 4, 0)),
              26: ((8, 2, 4, 0), (8, 2, 2, 0), (8, 2, 1, 1), (4, 4, 4, 0), (16, 1, 4, 0)),
              50: ((8, 4, 1, 0), (8, 4, 2, 0), (8, 4, 1, 1), (16, 2, 1, 0), (16, 2, 2, 0),
                   (16, 2, 1, 1), (4, 8, 1, 0), (4, 8, 2, 0)),
              98: ((16, 4, 1, 0), (16, 4, 2, 0), (8, 8, 1, 0), (8, 8, 2, 0), (32, 2, 1, 0)),
              202: ((32, 4, 1, 0),)}
    for C, shp in shapes.items():
        x = np.empty((3001, C), np.float32)
        tensor.fill_normal_array(x, C, 4.0)
        x[7, 1] = -500.0
        ref = oracle.softmax_ref(x)
        if C <= 128:
            assert "vec=2" in gu.plan(3001, C), gu.plan(3001, C)
        _native.set_tuning("vec2_max", 256)
        for lpr, nv, u, pf in shp:
            _native.set_tuning("k1_lpr", lpr)
            _native.set_tuning("k1_nv", nv)
            _native.set_tuning("k1_u", u)
            _native.set_tuning("k1_pf", pf)
            assert f"vec=2 lpr={lpr} nv={nv} u={u}" in gu.plan(3001, C)
            y, _ = gu.softmax_abi(x, 0)
            assert_parity(oracle, y, ref, what=(C, lpr, nv, u, pf))
        for k in ("k1_lpr", "k1_nv", "k1_u"):
            _native.set_tuning(k, 0)
        _native.set_tuning("k1_pf", -1)
        _native.set_tuning("vec2_max", 0)
        assert "vec=1" in gu.plan(3001, C)
        y, _ = gu.softmax_abi(x, 0)
        assert_parity(oracle, y, ref, what=(C, "32-bit"))
        _native.set_tuning("vec2_max", 128)


@pytest.mark.parametrize("C", [3, 5, 8, 10, 13, 18, 20, 25, 26, 36, 48, 50, 64, 63, 75, 98, 126, 127])
def test_k1_short_rows_job_size_keeps_bits(C, oracle):
    """Short rows: the K1 shape is a function of C, while rows per lane group,
    prefetch and the persistent grid follow the job size -- a large job
    (>= 4 Mi elements) and a small row block of it must give the same bits,
    and both match the oracle."""
    from paper_1904_12380_b200 import tensor

    rows = (1 << 22) // C + 777
    x = np.empty((rows, C), np.float32)
    tensor.fill_normal_array(x, C + 5, 4.0)
    x[3, C // 2] = -300.0
    big_plan, small_plan = gu.plan(rows, C), gu.plan(999, C)
    key = lambda p: p.split(" u=")[0]  # noqa: E731 -- vec / lpr / nv
    assert key(big_plan) == key(small_plan), (big_plan, small_plan)
    whole, bad = gu.softmax_abi(x, 0)
    assert bad == gu.NO_BAD
    part, _ = gu.softmax_abi(x[rows - 999:], 0)
    assert np.array_equal(part.view(np.uint32), whole[rows - 999:].view(np.uint32)), (big_plan, small_plan)
    idx = np.r_[0:2000, rows - 2000:rows]
    assert_parity(oracle, whole[idx], oracle.softmax_ref(x[idx]), what=(C, big_plan))


@pytest.mark.parametrize("rows,C", [(300, 2048), (37, 1536), (4096, 3072), (5, 2052),
                                    (2000, 1028), (1, 3072)])
def test_k1_medium_rows(rows, C, oracle):
    """128-bit rows of 1025..3072 floats: a whole warp holds the row in
    registers (K1, 16/24 vectors per lane); small jobs shrink the block so
    they spread over the SMs (same bits).  Clip firing, large negative row,
    strided pitch, non-finite detection."""
    from paper_1904_12380_b200 import tensor

    x = np.empty((rows, C), np.float32)
    tensor.fill_normal_array(x, C + rows, 5.0)
    x[0, C // 2] = -300.0
    x[rows // 2, :] -= 500.0
    plan = gu.plan(rows, C)
    assert plan.startswith("k1 vec=4 lpr=32"), plan
    for mode in (0, 1):
        ref = oracle.softmax_ref(x, clip=(mode == 0))
        y, bad = gu.softmax_abi(x, mode)
        assert bad == gu.NO_BAD
        assert_parity(oracle, y, ref, what=(rows, C, mode, plan))
    y, _ = gu.softmax_abi(x, 0, ldx=C + 8, ldy=C + 4)
    assert_parity(oracle, y, oracle.softmax_ref(x), what=(rows, C, "strided"))
    whole, _ = gu.softmax_abi(x, 0)
    part, _ = gu.softmax_abi(x[rows // 3:], 0)   # a row block: same bits
    assert np.array_equal(part.view(np.uint32), whole[rows // 3:].view(np.uint32))
    x2 = x.copy()
    x2[rows - 1, C - 1] = np.nan
    assert gu.softmax_abi(x2, 0)[1] == rows - 1


@pytest.mark.parametrize("rows,C", [(300, 8192), (4096, 4000), (2048, 5000), (64, 6144),
                                    (3, 8192), (1000, 3076), (4096, 5001), (300, 8191),
                                    (2000, 1283), (7, 3001), (513, 4097), (64, 6143),
                                    (300, 12288), (37, 16384), (1000, 10000), (129, 12289),
                                    (64, 16383), (5, 9001), (2, 16384)])
def test_k1m_medium_rows(rows, C, oracle):
    """Rows held in the registers of 2-8 warps (K1m): 128-bit rows of
    3073..16384 floats and rows of any length (32-bit accesses) from 1025 up --
    every mode, clip firing, a large negative row, strided pitch, row blocks
    bit-identical to the whole matrix, non-finite detection."""
    from paper_1904_12380_b200 import tensor

    x = np.empty((rows, C), np.float32)
    tensor.fill_normal_array(x, 3 * C + rows, 5.0)
    x[0, C - 1] = -300.0
    x[rows // 2, :] -= 500.0
    plan = gu.plan(rows, C)
    assert plan.startswith("k1m "), plan
    for mode in (0, 1, 2):
        ref = oracle.softmax_ref(x, clip=(mode == 0))
        y, bad = gu.softmax_abi(x, mode)
        assert bad == gu.NO_BAD
        assert_parity(oracle, y, ref, approx=(mode == 2), what=(rows, C, mode, plan))
    y, _ = gu.softmax_abi(x, 0, ldx=C + 12, ldy=C + 4)
    assert_parity(oracle, y, oracle.softmax_ref(x), what=(rows, C, "strided"))
    y, _ = gu.softmax_abi(x, 0, x_offset=1, y_offset=3, ldx=C + 3, ldy=C + 1)
    assert_parity(oracle, y, oracle.softmax_ref(x), what=(rows, C, "unaligned"))
    whole, _ = gu.softmax_abi(x, 0)
    part, _ = gu.softmax_abi(x[rows // 3:], 0)
    assert np.array_equal(part.view(np.uint32), whole[rows // 3:].view(np.uint32))
    x2 = x.copy()
    x2[rows - 1, 5] = np.inf
    assert gu.softmax_abi(x2, 0)[1] == rows - 1


@pytest.mark.parametrize("rows,C", [(2000, 1025), (300, 1151), (37, 1153), (5, 1279), (4100, 1280)])
def test_k1_one_warp_32bit_rows(rows, C, oracle):
    """32-bit rows of 1025..1280 floats held by one warp (K1, 36 / 40 floats per
    lane): every mode, clip firing, strided / unaligned views, row blocks
    bit-identical to the whole matrix, non-finite detection."""
    from paper_1904_12380_b200 import tensor

    x = np.empty((rows, C), np.float32)
    tensor.fill_normal_array(x, 5 * C + rows, 5.0)
    x[0, C - 1] = -300.0
    x[rows // 2, :] -= 500.0
    plan = gu.plan(rows, C)
    assert plan.startswith("k1 ") and "lpr=32" in plan, plan
    for mode in (0, 1, 2):
        ref = oracle.softmax_ref(x, clip=(mode == 0))
        y, bad = gu.softmax_abi(x, mode)
        assert bad == gu.NO_BAD
        assert_parity(oracle, y, ref, approx=(mode == 2), what=(rows, C, mode, plan))
    y, _ = gu.softmax_abi(x, 0, x_offset=1, y_offset=3, ldx=C + 3, ldy=C + 1)
    assert_parity(oracle, y, oracle.softmax_ref(x), what=(rows, C, "unaligned"))
    whole, _ = gu.softmax_abi(x, 0)
    part, _ = gu.softmax_abi(x[rows // 3:], 0)
    assert np.array_equal(part.view(np.uint32), whole[rows // 3:].view(np.uint32))
    x2 = x.copy()
    x2[rows - 1, 5] = np.nan
    assert gu.softmax_abi(x2, 0)[1] == rows - 1


def test_k1m_instantiations_and_k2_fallback(oracle):
    """Every K1m (warps per row, vectors per lane) shape that covers the row,
    and the TMA block-per-row K2 / K3g (k1m off) on the same rows -- including
    6144 columns, where K2 needs exactly 48 KB of dynamic shared memory."""
    from paper_1904_12380_b200 import tensor

    for C in (4096, 6144, 8192, 12288, 16384):
        x = np.empty((40, C), np.float32)
        tensor.fill_normal_array(x, C, 4.0)
        ref = oracle.softmax_ref(x)
        try:
            for wpr, nv in ((2, 16), (4, 8), (4, 12), (4, 16), (8, 8), (8, 12), (8, 16)):
                if wpr * 32 * nv * 4 < C:
                    continue
                _native.set_tuning("k1m_wpr", wpr)
                _native.set_tuning("k1m_nv", nv)
                y, _ = gu.softmax_abi(x, 0)
                assert_parity(oracle, y, ref, what=(C, wpr, nv))
            _native.set_tuning("k1m_wpr", 0)
            _native.set_tuning("k1m", 0)
            # k1m off: K2 up to 8192 columns; beyond, what took 8193..16384 before
            # K1m did (K3g, or the split latency path for a 40-row job)
            plan = gu.plan(40, C)
            assert plan.startswith("k2_tma") if C <= 8192 else plan.startswith(("k3_gres ", "k4_split")), plan
            y, _ = gu.softmax_abi(x, 0)
            assert_parity(oracle, y, ref, what=(C, "k1m off"))
        finally:
            _native.set_tuning("k1m", 1)
            _native.set_tuning("k1m_wpr", 0)
            _native.set_tuning("k1m_nv", 0)


@pytest.mark.parametrize("impl", ["g", "c", "c1x", "split"])
def test_every_long_row_kernel(impl, oracle):
    """Long-row kernels on the same ragged rows (last slice partial, clip
    firing): K3g grid-resident rows (g), K3c cluster-resident rows with two
    exchanges (c) or one (c1x), and the split path (K4) -- all against the
    oracle."""
    x = configs.generate("c4", 0, 40)[:, :200_004].copy()
    x[3, 777] = -500.0
    ref = oracle.softmax_ref(x)
    try:
        if impl == "g":
            _native.set_tuning("gres", 2)
        elif impl in ("c", "c1x"):
            _native.set_tuning("k3_impl", 5)
            _native.set_tuning("cluster_onex", 1 if impl == "c1x" else 0)
        else:
            _native.set_tuning("path", 2)
        plan = gu.plan(*x.shape)
        assert plan.split()[0] == {"g": "k3_gres", "c": "k3_cluster", "c1x": "k3_cluster",
                                   "split": "k4_split"}[impl], plan
        y, bad = gu.softmax_abi(x, 0)
        assert bad == gu.NO_BAD
        assert_parity(oracle, y, ref, what=(impl, plan))
    finally:
        _native.set_tuning("gres", 1)
        _native.set_tuning("k3_impl", 3)
        _native.set_tuning("cluster_onex", 0)
        _native.set_tuning("path", -1)


@pytest.mark.parametrize("P,st,split", [(2, 0, -1), (3, 2, 1), (10, 0, 1), (14, 3, -1), (14, 3, 1),
                                        (37, 4, -1), (37, 4, 0), (74, 5, -1), (74, 5, 0),
                                        (148, 0, -1)])
def test_k3_gres_group_sizes(P, st, split, oracle):
    """K3g with P CTAs per row and ring depth st (lag st-2: 1..3) -- ragged last
    slice, one- to many-group grids, more groups than rows, clip firing, a large
    negative row -- every mode."""
    C = 200_004 if P >= 10 else 30_004
    rows = 13
    x = configs.generate("c4", 0, rows)[:, :C].copy()
    x[3, 777] = -500.0
    x[5, :] -= 400.0
    _native.set_tuning("gres", 2)
    _native.set_tuning("gres_p", P)
    _native.set_tuning("gres_st", st)
    _native.set_tuning("gres_split", split)
    try:
        assert gu.plan(rows, C).startswith("k3_gres nseg=%d " % P), gu.plan(rows, C)
        if st:
            assert "stages=%d " % st in gu.plan(rows, C)
        for mode in (0, 1, 2):
            ref = oracle.softmax_ref(x, clip=(mode == 0))
            y, bad = gu.softmax_abi(x, mode)
            assert bad == gu.NO_BAD
            assert_parity(oracle, y, ref, approx=(mode == 2), what=(P, mode, gu.plan(rows, C)))
        x2 = x.copy()
        x2[9, C - 1] = np.inf
        x2[7, 0] = np.nan
        assert gu.softmax_abi(x2, 0)[1] == 7
    finally:
        _native.set_tuning("gres", 1)
        _native.set_tuning("gres_p", 0)
        _native.set_tuning("gres_st", 0)
        _native.set_tuning("gres_split", -1)


@pytest.mark.parametrize("P,st,lag,split", [(14, 3, 1, -1), (37, 8, 3, -1), (37, 6, 1, -1),
                                            (37, 6, 1, 1), (24, 5, 2, -1), (74, 8, 2, 0),
                                            (148, 8, 3, -1), (20, 4, 1, 1)])
def test_k3_gres_lag_depth_decoupled(P, st, lag, split, oracle):
    """K3g with the lag (rows between a row's local and output pass) set apart
    from the ring depth: st - lag - 1 rows load ahead.  Many row steps per
    group (so every ring slot and barrier id rotates several times), a ragged
    last slice, clip firing, every mode; plus a non-finite row."""
    C = 120_004
    rows = (148 // P) * 5 + 7 if P < 148 else 23
    x = configs.generate("c4", 1, rows)[:, :C].copy()
    x[2, 1234] = -500.0
    x[rows - 1, :] -= 400.0
    _native.set_tuning("gres", 2)
    _native.set_tuning("gres_p", P)
    _native.set_tuning("gres_st", st)
    _native.set_tuning("gres_lag", lag)
    _native.set_tuning("gres_split", split)
    try:
        plan = gu.plan(rows, C)
        assert plan.startswith("k3_gres nseg=%d " % P), plan
        assert "stages=%d " % st in plan and plan.endswith(" lag=%d" % lag), plan
        for mode in (0, 1, 2):
            ref = oracle.softmax_ref(x, clip=(mode == 0))
            y, bad = gu.softmax_abi(x, mode)
            assert bad == gu.NO_BAD
            assert_parity(oracle, y, ref, approx=(mode == 2), what=(P, st, lag, mode, plan))
        x2 = x.copy()
        x2[rows - 2, 17] = -np.inf
        x2[rows - 3, C - 2] = np.nan
        assert gu.softmax_abi(x2, 0)[1] == rows - 3
    finally:
        _native.set_tuning("gres", 1)
        _native.set_tuning("gres_p", 0)
        _native.set_tuning("gres_st", 0)
        _native.set_tuning("gres_lag", 0)
        _native.set_tuning("gres_split", -1)


def test_k3_gres_full_c4_rowsums():
    """K3g over all of c4 (1024 x 262144): every row sums to 1, determinism."""
    t = gu.torch()
    xd = t.from_numpy(configs.generate("c4")).cuda()
    _native.set_tuning("gres", 2)
    try:
        y1 = sk.softmax(xd, sk.KernelVariant.REFERENCE_CLIPPED)
        y2 = sk.softmax(xd, sk.KernelVariant.REFERENCE_CLIPPED)
        t.cuda.synchronize()
    finally:
        _native.set_tuning("gres", 1)
    assert bool(t.equal(y1, y2))
    rs = y1.double().sum(dim=1)
    assert float((rs - 1).abs().max()) <= 1e-5


@pytest.mark.parametrize("C", [4_194_304, 4_400_000, 8_000_000])
def test_rows_at_and_beyond_chip_capacity(C, oracle):
    """4 M floats: K3g at its largest group (148 CTAs, 2-stage ring).  Longer
    rows than the chip's shared memory holds (> 148 x 225 KB / 2 stages) fall
    back to the split path; all match the oracle."""
    from paper_1904_12380_b200 import tensor

    x = np.empty((3, C), np.float32)
    tensor.fill_normal_array(x, 17, 3.0)
    x[1, C // 3] = -400.0
    fits = C <= 148 * 28_800
    _native.set_tuning("gres", 2 if fits else 1)  # 3 rows alone would take the latency path
    try:
        plan = gu.plan(3, C)
        assert ("k3_gres" in plan) == fits, plan
        y, bad = gu.softmax_abi(x, 0)
    finally:
        _native.set_tuning("gres", 1)
    assert bad == gu.NO_BAD
    assert_parity(oracle, y, oracle.softmax_ref(x, True, nthreads=0), what=plan)


@pytest.mark.parametrize("rows,C", [(200, 50257), (40, 262147), (8, 1_000_003), (600, 16385),
                                    (300, 20001)])
def test_k3g_unaligned_rows(rows, C, oracle):
    """Rows of any length / alignment past one CTA: K3g cuts each row's
    slices at x's 16-B boundaries, stages them by TMA and reads the <= 3 head
    / tail floats from global memory -- every mode, clip, unaligned bases and
    pitches (y in and out of x's phase), non-finite detection, determinism."""
    from paper_1904_12380_b200 import tensor

    x = np.empty((rows, C), np.float32)
    tensor.fill_normal_array(x, C % 1000 + rows, 4.0)
    x[0, 1] = -400.0
    x[rows - 1, C - 1] = 30.0
    plan = gu.plan(rows, C)
    assert plan.startswith("k3_gres_unal"), plan
    for mode in (0, 1, 2):
        ref = oracle.softmax_ref(x, clip=(mode == 0))
        y, bad = gu.softmax_abi(x, mode)
        assert bad == gu.NO_BAD
        assert_parity(oracle, y, ref, approx=(mode == 2), what=(rows, C, mode, plan))
    ref = oracle.softmax_ref(x)
    for xo, yo, ldx, ldy in ((1, 0, C + 3, C + 1), (3, 2, C + 1, C + 6), (2, 2, C + 2, C + 2)):
        y, _ = gu.softmax_abi(x, 0, x_offset=xo, y_offset=yo, ldx=ldx, ldy=ldy)
        assert_parity(oracle, y, ref, what=(rows, C, xo, yo, ldx, ldy))
    y1, _ = gu.softmax_abi(x, 0)
    y2, _ = gu.softmax_abi(x, 0)
    assert np.array_equal(y1.view(np.uint32), y2.view(np.uint32))
    x2 = x.copy()
    x2[rows // 2, C // 2] = np.nan
    assert gu.softmax_abi(x2, 0)[1] == rows // 2


# ---------------------------------------------------------------- errors / faults
@pytest.mark.parametrize("C", [50, 128, 1000, 4097, 8192, 70000])
def test_nonfinite_reports_first_bad_row(C):
    rows = 40
    x = np.ones((rows, C), np.float32)
    x[31, C - 1] = np.inf
    x[17, C // 2] = np.nan
    x[25, 0] = -np.inf
    _, bad = gu.softmax_abi(x, 0)
    assert bad == 17, gu.plan(rows, C)
    t = gu.torch()
    with pytest.raises(sk.NumericDomainError, match="row 17"):
        sk.softmax(t.from_numpy(x).cuda(), sk.KernelVariant.REFERENCE_CLIPPED)
    with pytest.raises(sk.NumericDomainError, match="row 17"):
        sk.softmax(sk.Matrix2D.from_array(x), sk.KernelVariant.REFERENCE_CLIPPED)
    # the flag was reset: a clean call succeeds afterwards
    sk.softmax(t.ones(3, C, device="cuda"), sk.KernelVariant.REFERENCE_CLIPPED)


def test_skip_max_shift_fault_is_caught(oracle):
    """kernels._SKIP_MAX_SHIFT (reference kernels.py:103-105): without the max
    shift, large logits overflow and the parity harness must FAIL."""
    from paper_1904_12380_b200 import kernels

    x = configs.generate("c1") + np.float32(80.0)
    ref = oracle.softmax_ref(x)
    t = gu.torch()
    kernels._SKIP_MAX_SHIFT = True
    try:
        y = sk.softmax(t.from_numpy(x).cuda(), sk.KernelVariant.REFERENCE_CLIPPED).cpu().numpy()
    finally:
        kernels._SKIP_MAX_SHIFT = False
    assert not oracle.parity(y, ref)["ok"]
    y = sk.softmax(t.from_numpy(x).cuda(), sk.KernelVariant.REFERENCE_CLIPPED).cpu().numpy()
    assert oracle.parity(y, ref)["ok"]


# ---------------------------------------------------------------- invariants
@pytest.mark.parametrize("rows,C,kind", [(1, 32000, "k3_cluster"), (8, 50257, "k4_split"),
                                         (3, 262144, "k4_split"), (2, 65536, "k3_cluster"),
                                         (32, 151936, "k4_split"), (512, 262144, "k3_gres")])
def test_small_batches_wide_rows(rows, C, kind, oracle):
    """Decode-sized batches over wide rows: with <= 3 row steps per K3g group
    the latency path is taken (cluster kernel for 1-2 rows, split otherwise);
    larger jobs keep K3g -- all matching the oracle."""
    from paper_1904_12380_b200 import tensor

    x = np.empty((rows, C), np.float32)
    tensor.fill_normal_array(x, C + 17 * rows, 3.0)
    x[0, C // 3] = 25.0
    plan = gu.plan(rows, C)
    assert plan.startswith(kind), plan
    for mode in (0, 1):
        y, bad = gu.softmax_abi(x, mode)
        assert bad == gu.NO_BAD
        assert_parity(oracle, y, oracle.softmax_ref(x, clip=(mode == 0)), what=(rows, C, plan))


def test_shift_invariance_and_order():
    x = configs.generate("c3", 0, None)[:256]
    base, _ = gu.softmax_abi(x)
    for c in (-50.0, -1.0, 1.0, 50.0):
        y, _ = gu.softmax_abi(x + np.float32(c))
        assert np.max(np.abs(y - base)) <= 1e-6
    ranks_in = np.argsort(np.argsort(x[:8], axis=1, kind="stable"), axis=1)
    y8 = base[:8]
    # order preserved where inputs are distinct (ties/clip floor aside)
    for r in range(8):
        ux = x[r] > x[r].max() - 60
        assert np.all(np.diff(y8[r][ux][np.argsort(x[r][ux])]) >= 0)
    del ranks_in


def test_deterministic_and_row_shard_bitwise():
    """Same bits run to run, and a row block computed alone equals the same
    rows of the whole matrix (row sharding needs no communication)."""
    for name, split in (("c2", 20000), ("c1", 1024), ("c3", 4096)):
        x = configs.generate(name)
        y1, _ = gu.softmax_abi(x)
        y2, _ = gu.softmax_abi(x)
        assert np.array_equal(y1.view(np.uint32), y2.view(np.uint32))
        a, _ = gu.softmax_abi(x[:split])
        b, _ = gu.softmax_abi(x[split:])
        assert np.array_equal(np.concatenate([a, b]).view(np.uint32), y1.view(np.uint32))
    spec = configs.get("c4")
    x = configs.generate(spec, 0, 64)  # c4 sharded 8 ways
    y, _ = gu.softmax_abi(x)
    a, _ = gu.softmax_abi(x[5:45])  # a 40-row block: same (row-length-only) plan
    assert gu.plan(40, spec.cols).split(" grid=")[0] == gu.plan(64, spec.cols).split(" grid=")[0]
    assert gu.plan(40, spec.cols).startswith("k3_gres")
    assert np.array_equal(a.view(np.uint32), y[5:45].view(np.uint32))


@pytest.mark.parametrize("name", ["c4"])
def test_host_path_chunks_keep_device_bits(name):
    """The host-buffer pipeline splits a long-row job into small row chunks;
    each chunk takes the job's throughput plan (not the latency path a small
    standalone call would take), so the result is bit-identical to the
    device path on the whole matrix."""
    spec = configs.get(name)
    x = configs.generate(spec, 0, 96)
    dev, _ = gu.softmax_abi(x)
    _native.set_tuning("host_chunk_kb", 4096)  # 4-row chunks
    try:
        m = sk.Matrix2D.from_array(x, pinned=True)
        out = sk.softmax(m, sk.KernelVariant.REFERENCE_CLIPPED)
    finally:
        _native.set_tuning("host_chunk_kb", 0)
    assert np.array_equal(out.view2d.view(np.uint32), dev.view(np.uint32))


def test_host_path_equals_device_path():
    x = configs.generate("c3")
    dev, _ = gu.softmax_abi(x)
    m = sk.Matrix2D.from_array(x, pinned=True)
    out = sk.softmax(m, sk.KernelVariant.REFERENCE_CLIPPED)
    assert np.array_equal(out.view2d.view(np.uint32), dev.view(np.uint32))
    pageable = sk.softmax(sk.Matrix2D.from_array(x), sk.KernelVariant.REFERENCE_CLIPPED)
    assert np.array_equal(pageable.view2d.view(np.uint32), dev.view(np.uint32))
    arr = sk.softmax(x, sk.KernelVariant.REFERENCE_CLIPPED)
    assert np.array_equal(arr.view(np.uint32), dev.view(np.uint32))
    _native.set_tuning("host_zero_copy", 1)
    try:
        zc = sk.softmax(m, sk.KernelVariant.REFERENCE_CLIPPED)
        assert np.array_equal(zc.view2d.view(np.uint32), dev.view(np.uint32))
    finally:
        _native.set_tuning("host_zero_copy", 0)
    for kb in (256, 1024):  # many chunks: ring reuse, ramp
        _native.set_tuning("host_chunk_kb", kb)
        try:
            ck = sk.softmax(m, sk.KernelVariant.REFERENCE_CLIPPED)
            assert np.array_equal(ck.view2d.view(np.uint32), dev.view(np.uint32))
        finally:
            _native.set_tuning("host_chunk_kb", 0)


@pytest.mark.parametrize("kb,threads", [(0, 0), (256, 0), (1024, 1), (512, 3)])
def test_host_path_pageable_staging(kb, threads):
    """Pageable caller buffers (the reference's np.zeros Matrix2D) go through
    page-locked staging slots copied by the host thread pool: every mix of
    pageable / pinned input and output, many chunks (staging-ring reuse), any
    thread count -- bit-identical to the device path."""
    x = configs.generate("c3")
    dev, _ = gu.softmax_abi(x)
    _native.set_tuning("host_chunk_kb", kb)
    _native.set_tuning("host_threads", threads)
    try:
        for pin_in in (False, True):
            for pin_out in (False, True):
                m = sk.Matrix2D.from_array(x, pinned=pin_in)
                o = sk.alloc_matrix(*x.shape, pinned=pin_out)
                sk.softmax(m, sk.KernelVariant.REFERENCE_CLIPPED, out=o)
                assert np.array_equal(o.view2d.view(np.uint32), dev.view(np.uint32)), \
                    (kb, threads, pin_in, pin_out)
    finally:
        _native.set_tuning("host_chunk_kb", 0)
        _native.set_tuning("host_threads", 0)


def test_every_variant_through_public_api(oracle):
    x = configs.generate("c2", 0, 512)
    t = gu.torch()
    xd = t.from_numpy(x).cuda()
    for v in sk.LADDER:
        y = sk.softmax(xd, v).cpu().numpy()
        ref = oracle.softmax_ref(x, clip=(v is sk.KernelVariant.REFERENCE_CLIPPED))
        assert_parity(oracle, y, ref, approx=(v is sk.KernelVariant.FULL_VECTORIZED_APPROX_EXP),
                      what=v)


# ---------------------------------------------------------------- exp accuracy
def test_exp_accuracy_exhaustive():
    """Every fp32 in [-64, 0] (the ValueClip range; ~1.1e9 values) and in
    [-88, -64] through the kernels' exponential vs the double exp.  The
    reference's glibc expf is within 0.5 ulp, so kernel-vs-reference per-element
    differences are bounded by max_ulp + 0.5 (SPEC.md:146-147 examples)."""
    import ctypes

    L = _native.lib()
    for mode, lo, hi, ulp_bound in ((0, -64.0, 0.0, 3.0), (1, -87.0, 0.0, 3.0),
                                    (2, -87.0, 0.0, 200.0)):
        u = ctypes.c_double()
        r = ctypes.c_double()
        _native.check(L.sk_exp_accuracy(mode, lo, hi, ctypes.byref(u), ctypes.byref(r), 0))
        print(f"mode {mode} [{lo}, {hi}]: max {u.value:.3f} ulp, max rel {r.value:.3e}")
        assert u.value <= ulp_bound, (mode, u.value)
        if mode == 2:
            assert r.value <= 1e-5  # FullVectorizedApproxExp tolerance, bench.py:52


def test_device_api_argument_errors():
    """softmax / softmax_into on CUDA tensors reject what the kernels cannot
    read: non-unit column stride (a single-row view too), wrong dtype / rank /
    device, mismatched shapes -- as ArgumentError, like the reference."""
    t = gu.torch()
    x = t.randn(4, 64, device="cuda")
    for bad in (x[:, ::2], x[0:1, ::2], x.t(), x.double(), x[0], x.cpu()):
        with pytest.raises(sk.ArgumentError):
            sk.softmax(bad, sk.KernelVariant.REFERENCE_CLIPPED)
    with pytest.raises(sk.ArgumentError):
        sk.softmax_into(x, t.empty(4, 65, device="cuda"), sk.KernelVariant.REFERENCE_CLIPPED)
    y = sk.softmax(x[1:3, 8:40], sk.KernelVariant.REFERENCE_CLIPPED)  # strided rows are fine
    assert t.allclose(y, t.softmax(x[1:3, 8:40], dim=1), atol=1e-6)


def test_concurrent_streams_long_rows(oracle):
    """K3g is a cooperative grid that spins on its groups' exchanges: several
    streams launching it concurrently (and a K1 job beside them) must neither
    deadlock nor corrupt each other -- each launch's CTAs are co-resident by
    construction and each stream has its own exchange block."""
    t = gu.torch()
    x1 = t.from_numpy(configs.generate("c4", 0, 64)).cuda()
    x2 = t.from_numpy(configs.generate("c4", 64, 64)).cuda()
    x3 = t.from_numpy(configs.generate("c2", 0, 8192)).cuda()
    ys = [t.empty_like(x) for x in (x1, x2, x3)]
    streams = [t.cuda.Stream() for _ in range(3)]
    _native.set_tuning("gres_timeout_spins", 1 << 20)  # a deadlock would abort, not hang
    try:
        for _ in range(20):
            for x, y, s in zip((x1, x2, x3), ys, streams):
                with t.cuda.stream(s):
                    sk.softmax_into(x, y, sk.KernelVariant.REFERENCE_CLIPPED, check_finite=False)
        t.cuda.synchronize()
        from paper_1904_12380_b200.kernels import check_device_flag

        check_device_flag()  # raises on an aborted exchange
    finally:
        _native.set_tuning("gres_timeout_spins", 0)
    for x, y in zip((x1, x2, x3), ys):
        ref = oracle.softmax_ref(x.cpu().numpy(), True, nthreads=0)
        assert oracle.parity(y.cpu().numpy(), ref)["ok"]
