"""CPU tests of the host side: generators pinned to the reference, the
Matrix2D / KernelVariant / LaneConfig mirror, the C ABI's exported symbols
and argument checks (no kernel launches: there is no GPU here)."""

import ctypes
import re

import numpy as np
import pytest

import paper_1904_12380_b200 as sk
from paper_1904_12380_b200 import configs, tensor
from tests.conftest import ROOT


# ------------------------------------------------------------ generators
def test_fill_uniform_bit_identical_to_reference(golden, golden_meta):
    for f in golden_meta["fill_uniform"]:
        m = tensor.alloc_matrix(1, f["n"])
        tensor.fill_uniform(m, tensor.FillSpec(f["seed"], f["low"], f["high"]))
        assert np.array_equal(m.data[:64], golden[f"fill/{f['seed']}/prefix"])
        assert configs.sha256(m.data) == f["sha256"]


def test_generators_chunk_independent():
    full = np.empty(10_001, np.float32)
    tensor.fill_normal_array(full, 5, 2.0)
    for a, b in ((0, 3), (3, 4097), (4097, 10_001), (1, 2)):
        part = np.empty(b - a, np.float32)
        tensor.fill_normal_array(part, 5, 2.0, start=a)
        assert np.array_equal(part, full[a:b]), (a, b)
    u = np.empty(9999, np.float32)
    tensor.fill_uniform_array(u, 1, -10, 10)
    part = np.empty(5000, np.float32)
    tensor.fill_uniform_array(part, 1, -10, 10, start=4999)
    assert np.array_equal(part, u[4999:])


def test_generators_thread_count_invariant():
    a = np.empty(300_000, np.float32)
    b = np.empty(300_000, np.float32)
    tensor.fill_normal_array(a, 3, 5.0, nthreads=1)
    tensor.fill_normal_array(b, 3, 5.0, nthreads=7)
    assert np.array_equal(a, b)


def test_normal_generator_statistics():
    a = np.empty(1 << 20, np.float32)
    tensor.fill_normal_array(a, 0, 4.0)
    assert abs(a.mean()) < 0.02
    assert abs(a.std() - 4.0) < 0.02


def test_config_inputs_match_recorded_hashes(golden_meta):
    for name in ("c1", "c2", "c3"):
        assert configs.sha256(configs.generate(name)) == golden_meta["configs"][name]["input_sha256"]


def test_c3_plants_exactly_one_percent():
    x = configs.generate("c3")
    assert int(np.count_nonzero(x == -100.0)) == 81_920


def test_row_range_generation_matches_whole():
    spec = configs.get("c4")
    a = configs.generate(spec, row_start=5, row_count=2)
    b = np.empty((2, spec.cols), np.float32)
    tensor.fill_normal_array(b, spec.seed, spec.sigma, start=5 * spec.cols)
    assert np.array_equal(a, b)
    with pytest.raises(sk.ArgumentError):
        configs.generate("c3", row_start=1, row_count=1)


# ------------------------------------------------------------ mirror types
def test_matrix2d_validation_mirrors_reference():
    with pytest.raises(sk.ArgumentError):
        tensor.Matrix2D(0, 3, np.zeros(0, np.float32))
    with pytest.raises(sk.ArgumentError):
        tensor.Matrix2D(1, 3, np.zeros(3, np.float64))
    with pytest.raises(sk.ArgumentError):
        tensor.Matrix2D(1, 4, np.zeros(3, np.float32))
    raw = np.zeros(16, np.float32)
    off = 1 if raw.ctypes.data % 32 == 0 else 0
    with pytest.raises(sk.ArgumentError):
        tensor.Matrix2D(1, 4, raw[off:off + 4])
    m = tensor.alloc_matrix(3, 5)
    assert m.data.ctypes.data % 32 == 0 and m.shape == (3, 5)
    assert isinstance(sk.ArgumentError("x"), ValueError)
    assert isinstance(sk.ResourceError("x"), MemoryError)


def test_variants_and_modes():
    assert [v.value for v in sk.LADDER] == [
        "ReferenceClipped", "ReferenceInference", "MklStyleScalar", "VectorizedSum",
        "FullVectorized", "FullVectorizedApproxExp"]
    assert sk.KernelVariant.from_name("FullVectorized") is sk.KernelVariant.FULL_VECTORIZED
    with pytest.raises(sk.ArgumentError):
        sk.KernelVariant.from_name("nope")
    modes = [sk.variant_mode(v) for v in sk.LADDER]
    assert modes == [0, 1, 1, 1, 1, 2]
    with pytest.raises(sk.ArgumentError):
        sk.variant_mode("ReferenceClipped")
    assert sk.CLIP_FLOOR == np.float32(-64.0)
    assert sk.FLT_MIN_NORMAL == np.float32(np.finfo(np.float32).tiny)


def test_lane_config():
    assert sk.LaneConfig().width == 8 and sk.LaneConfig(16).half_width == 8
    for bad in (2, 6, 0):
        with pytest.raises(sk.ArgumentError):
            sk.LaneConfig(bad)


# ------------------------------------------------------------ C ABI
def _header_functions():
    text = (ROOT / "include" / "softmax_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sk_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol(native):
    names = _header_functions()
    assert len(names) >= 17
    L = native.lib()
    for n in names:
        assert hasattr(L, n), n
        assert n in native.SIGNATURES, f"{n} missing from the ctypes binding"


def test_abi_version_and_status_strings(native):
    L = native.lib()
    assert L.sk_abi_version() == 1
    assert L.sk_status_string(0) == b"ok"
    assert L.sk_status_string(2) == b"non-finite logits"


def test_argument_errors_need_no_gpu(native):
    L = native.lib()
    # cols < 1, ld < cols, bad mode: rejected before any CUDA call
    assert L.sk_softmax_f32(1, 2, 4, 0, 4, 4, 0, None, None, 0, None) == native.SK_ERR_ARGUMENT
    assert L.sk_softmax_f32(1, 2, 4, 8, 4, 8, 0, None, None, 0, None) == native.SK_ERR_ARGUMENT
    assert L.sk_softmax_f32(1, 2, 4, 8, 8, 8, 7, None, None, 0, None) == native.SK_ERR_ARGUMENT
    assert L.sk_softmax_f32(None, None, 0, 8, 8, 8, 0, None, None, 0, None) == native.SK_OK
    with pytest.raises(sk.ArgumentError):
        native.check(native.SK_ERR_ARGUMENT)
    with pytest.raises(sk.NumericDomainError):
        native.check(native.SK_ERR_NONFINITE)
    with pytest.raises(sk.ResourceError):
        native.check(native.SK_ERR_RESOURCE)
    assert L.sk_set_tuning(b"no_such_key", 1) == native.SK_ERR_ARGUMENT
    assert L.sk_fill_uniform_f32(None, 4, 1, 1.0, 0.0, 0, 1) == native.SK_ERR_ARGUMENT


def test_workspace_sizes(native):
    L = native.lib()
    assert L.sk_softmax_workspace_bytes(512, 262144) >= 512 * 32 * 16
    assert L.sk_row_stats_workspace_bytes(1024, 1 << 20) >= 1024 * 256 * 16


def test_product_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    m = tensor.alloc_matrix(2, 3)
    with pytest.raises(sk.SoftmaxKitError):
        sk.softmax(m, sk.KernelVariant.REFERENCE_CLIPPED)
    with pytest.raises(sk.ArgumentError):
        sk.softmax(torch.zeros(2, 3), sk.KernelVariant.REFERENCE_CLIPPED)  # CPU tensor


def test_product_never_imports_oracle():
    for p in (ROOT / "paper_1904_12380_b200").rglob("*.py"):
        src = p.read_text()
        assert "import oracle" not in src and "from oracle" not in src, p
    for p in (ROOT / "paper_1904_12380_b200" / "csrc").iterdir():
        assert "sk_oracle" not in p.read_text(), p


def test_torch_ops_register_without_a_gpu():
    """torch.ops.softmax_b200 loads on a CPU-only host; every op has a schema
    and only a CUDA kernel (a CPU tensor raises: no CPU fallback)."""
    import torch

    from paper_1904_12380_b200 import torch_ops

    ops = torch_ops.load()
    for name, schema in (("softmax_fwd", "softmax_fwd(Tensor x, bool clip) -> Tensor"),
                         ("softmax_fwd_out", "softmax_fwd_out(Tensor x, Tensor(a!) y, bool clip) -> ()"),
                         ("row_max", "row_max(Tensor x) -> Tensor"),
                         ("row_sumexp", "row_sumexp(Tensor x, Tensor gmax, bool clip) -> Tensor"),
                         ("normalize_", "normalize_(Tensor x, Tensor gmax, Tensor gsum, Tensor(a!) y, bool clip) -> ()")):
        op = getattr(ops, name)
        assert str(op.default._schema) == "softmax_b200::" + schema
    with pytest.raises((NotImplementedError, RuntimeError)):
        ops.softmax_fwd(torch.zeros(2, 3), True)


def test_generate_cols_matches_full_rows():
    """A column shard generated alone equals the same columns of the whole
    matrix (every rank of a column-sharded run builds its shard independently)."""
    spec = configs.InputSpec("t", 7, 1000, "normal", 3, sigma=2.0)
    full = configs.generate(spec)
    for c0, w in ((0, 250), (250, 250), (333, 1), (999, 1), (1, 998)):
        assert np.array_equal(configs.generate_cols(spec, c0, w), full[:, c0:c0 + w])
    u = configs.InputSpec("u", 3, 64, "uniform", 5, low=-1.0, high=1.0)
    assert np.array_equal(configs.generate_cols(u, 16, 32), configs.generate(u)[:, 16:48])
