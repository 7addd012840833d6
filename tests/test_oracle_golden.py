"""The C oracle is pinned bit-for-bit to the reference's own outputs
(tests/golden/*, produced by running /root/reference in the build container)."""

import numpy as np
import pytest


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


@pytest.mark.parametrize("case", ["spec_123", "spec_zeros", "spec_single", "spec_big", "spec_clip"])
def test_spec_known_answers_bit_exact(golden, oracle, case):
    x = golden[f"{case}/x"]
    for rung, clip in (("clipped", True), ("inference", False)):
        y = oracle.softmax_ref(x, clip)
        assert np.array_equal(bits(y), bits(golden[f"{case}/{rung}"])), (case, rung)


def test_spec_values(oracle):
    # SPEC.md:175-177, :523 and SURVEY §4 known answers
    y = oracle.softmax_ref(np.array([[1, 2, 3]], np.float32))
    np.testing.assert_allclose(y[0], [0.09003057, 0.24472847, 0.66524096], atol=1e-6)
    assert np.all(oracle.softmax_ref(np.zeros((1, 4), np.float32)) == 0.25)
    assert oracle.softmax_ref(np.array([[3.0]], np.float32))[0, 0] == 1.0
    x = np.array([[0.0, -100.0]], np.float32)
    assert oracle.softmax_ref(x, clip=True)[0, 1] > 0  # ValueClip keeps it positive
    assert oracle.softmax_ref(x, clip=False)[0, 1] == 0  # inference flushes to +0


def test_sweep_bit_exact(golden, golden_meta, oracle):
    for C in golden_meta["sweep"]:
        x = golden[f"sweep/{C}/x"]
        for rung, clip in (("clipped", True), ("inference", False)):
            y = oracle.softmax_ref(x, clip)
            assert np.array_equal(bits(y), bits(golden[f"sweep/{C}/{rung}"])), (C, rung)


def test_config_rows_bit_exact(golden, oracle):
    for name in ("c1", "c3"):
        y = oracle.softmax_ref(golden[f"{name}/x"], True)
        assert np.array_equal(bits(y), bits(golden[f"{name}/clipped"])), name


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_full_config_hash_matches_reference(golden_meta, oracle, name):
    from paper_1904_12380_b200 import configs

    meta = golden_meta["configs"][name]
    x = configs.generate(name)
    assert configs.sha256(x) == meta["input_sha256"]
    y = oracle.softmax_ref(x, True, nthreads=0)
    assert configs.sha256(y) == meta["ref_clipped_sha256"]


def test_multithreaded_oracle_is_bitwise_single_threaded(oracle):
    from paper_1904_12380_b200 import configs

    x = configs.generate("c1")
    a = oracle.softmax_ref(x, True, nthreads=1)
    b = oracle.softmax_ref(x, True, nthreads=0)
    assert np.array_equal(bits(a), bits(b))


def test_nonfinite_rejected_with_first_row(oracle):
    x = np.zeros((6, 5), np.float32)
    x[4, 2] = np.inf
    x[2, 0] = np.nan
    with pytest.raises(ValueError, match="row 2"):
        oracle.softmax_ref(x)


def test_lane_reductions_match_reference(golden, oracle):
    for W in (4, 8, 16):
        for n in (1, 3, 7, 11, 64, 515):
            a = golden[f"lanes/{W}/{n}/a"]
            assert oracle.lanes_max(a, W) == golden[f"lanes/{W}/{n}/max"][0]
            assert bits(oracle.lanes_sum(a, W)) == bits(golden[f"lanes/{W}/{n}/sum"][0])


def test_philox_matches_numpy(oracle):
    for seed, start, n in ((1, 0, 9), (7, 1001, 5), (123456789, 3, 17)):
        want = np.random.Philox(key=seed).random_raw(start + n)[start:]
        assert np.array_equal(oracle.philox_raw(seed, start, n), want)


def test_metrics():
    import oracle as o

    ref = np.array([[0.25, 0.75]])
    assert o.max_abs_err(ref, ref) == 0.0
    assert o.max_rel_err(np.array([[0.5, 0.5]]), ref) == pytest.approx(1.0)
    assert o.max_rowsum_dev(np.array([[0.5, 0.6]])) == pytest.approx(0.1)
    assert o.max_rel_err(np.array([[np.nan, 1.0]]), ref) == float("inf")
    assert o.max_rel_err(np.array([[1e-30, 1.0]]), np.array([[0.0, 1.0]])) == float("inf")
    # flush boundary (unclipped rungs): FLT_MIN within the relative tolerance
    # may land on either side of the y < FLT_MIN -> 0 flush
    fm = np.float32(1.1754943508222875e-38)
    assert o.max_rel_err(np.array([[fm, 1.0]]), np.array([[0.0, 1.0]])) == 0.0
    assert o.max_rel_err(np.array([[0.0, 1.0]]), np.array([[fm, 1.0]])) == 0.0
    assert o.max_rel_err(np.array([[fm * 1.001, 1.0]]), np.array([[0.0, 1.0]])) == float("inf")


def _component_rows(g):
    return sorted({k.split("/")[0] for k in g.files if k.endswith("/row")})


def test_component_ops_bit_exact(golden_components, oracle):
    """The oracle's restatement of the 1-D component operations
    (kernels.py:229-276) reproduces the reference's outputs bit for bit."""
    g = golden_components
    for x, y in zip(g["clip/x"], g["clip/y"]):
        assert bits(oracle.value_clip(x)) == bits(y)
    for name in _component_rows(g):
        r = g[f"{name}/row"]
        m = oracle.row_max_scalar(r)
        assert bits(m) == bits(g[f"{name}/max"][0]), name
        sh = oracle.subtract_broadcast(r, m)
        assert np.array_equal(bits(sh), bits(g[f"{name}/sub_max"])), name
        assert np.array_equal(bits(oracle.subtract_broadcast(r, 3.25)), bits(g[f"{name}/sub_325"]))
        e = oracle.exp_batch(sh)
        assert np.array_equal(bits(e), bits(g[f"{name}/exp"])), name
        s = oracle.row_sum_scalar(e)
        assert bits(s) == bits(g[f"{name}/sum_exp"][0]), name
        assert bits(oracle.row_sum_scalar(r)) == bits(g[f"{name}/sum_row"][0]), name
        assert np.array_equal(bits(oracle.scale_reciprocal(e, s)), bits(g[f"{name}/scaled"])), name
        st = oracle.row_stats(r)
        assert np.array_equal(bits(np.array(st, np.float32)), bits(g[f"{name}/stats"])), name


def test_oracle_config_table_matches_product():
    """oracle/inputs.py restates configs.py's table (same shapes, laws, seeds)."""
    import inputs

    from paper_1904_12380_b200 import configs

    assert set(inputs.CONFIGS) == set(configs.CONFIGS)
    for k, a in inputs.CONFIGS.items():
        b = configs.CONFIGS[k]
        assert (a.rows, a.cols, a.dist, a.seed, a.sigma, a.low, a.high, a.plant_count,
                a.plant_value) == (b.rows, b.cols, b.dist, b.seed, b.sigma, b.low, b.high,
                                   b.plant_count, b.plant_value), k
        assert a.describe() == b.describe()


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_oracle_generator_matches_recorded_inputs(golden_meta, name):
    """The checker's own generators rebuild the exact input bytes the reference
    outputs were recorded on (input SHA-256 in golden.json)."""
    import inputs

    assert inputs.sha256(inputs.generate(name)) == golden_meta["configs"][name]["input_sha256"]


def test_oracle_generator_row_blocks_match_product():
    import inputs

    from paper_1904_12380_b200 import configs

    for name, start, count in (("c5a", 12345, 77), ("c4", 3, 2), ("c5b", 1000, 1), ("c2", 7, 9)):
        a = inputs.generate(name, start, count)
        b = configs.generate(name, start, count)
        assert np.array_equal(bits(a), bits(b)), name


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c4", "c5a", "c5b"])
def test_full_big_config_hash_matches_reference(golden_meta, oracle, name):
    """Every output element of the big configs: the oracle's ReferenceClipped
    output hash equals the hash recorded by running the reference itself on the
    full config (tests/golden/make_golden.py); inputs from the checker's own
    generator, pinned to the recorded input hash."""
    import inputs

    meta = golden_meta["configs"][name]
    x = inputs.generate(name)
    assert inputs.sha256(x) == meta["input_sha256"]
    y = oracle.softmax_ref(x, True, nthreads=0)
    del x
    assert inputs.sha256(y) == meta["ref_clipped_sha256"]
