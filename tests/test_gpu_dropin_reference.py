"""Drop-in against the LIVE reference (softmax_kit from baseline/_ref, the
unmodified reference package): a caller that swaps only the ``softmax``
import keeps its own Matrix2D / KernelVariant / LaneConfig / error classes,
and INTEGRATION.md §3's ctypes stub, installed inside softmax_kit.kernels,
dispatches the reference's own entry point to the GPU."""

import ctypes
import types

import numpy as np
import pytest

import paper_1904_12380_b200 as sk
from paper_1904_12380_b200 import _native, configs
from tests import gpu_util as gu
from tests import refpkg

pytestmark = pytest.mark.gpu
REF = refpkg.load()
needs_ref = pytest.mark.skipif(REF is None, reason="baseline/_ref (softmax_kit) not installed")


def _ref_matrix(x):
    m = REF.tensor.alloc_matrix(*x.shape)
    m.view2d[:] = x
    return m


@needs_ref
@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_swap_only_the_softmax_import(name, oracle):
    """softmax(reference Matrix2D, reference KernelVariant, reference
    LaneConfig) returns the reference's Matrix2D class, within the north-star
    gate of the live reference's own output, and bit-identical to the device
    path."""
    x = configs.generate(name)
    m = _ref_matrix(x)
    V = REF.kernels.KernelVariant
    live = REF.kernels.softmax(m, V.REFERENCE_CLIPPED)           # the reference, on the CPU
    ours = sk.softmax(m, V.REFERENCE_CLIPPED, REF.simd_reduce.LaneConfig())
    assert type(ours) is type(m)
    assert ours.shape == m.shape and ours.data.ctypes.data % 32 == 0
    d = oracle.parity(ours.view2d, live.view2d)
    assert d["ok"], (name, d)
    dev, _ = gu.softmax_abi(x)
    assert np.array_equal(ours.view2d.view(np.uint32), dev.view(np.uint32))
    # the reference's input is untouched (kernels.py:350-362 never mutates m)
    assert np.array_equal(m.view2d.view(np.uint32), x.view(np.uint32))


@needs_ref
def test_nonfinite_raises_the_reference_error_class():
    x = configs.generate("c1")
    x[37, 5] = np.nan
    x[900, 0] = np.inf
    m = _ref_matrix(x)
    with pytest.raises(REF.errors.NumericDomainError, match="row 37"):
        sk.softmax(m, REF.kernels.KernelVariant.REFERENCE_CLIPPED)
    with pytest.raises(REF.errors.NumericDomainError, match="row 37"):
        REF.kernels.softmax(m, REF.kernels.KernelVariant.REFERENCE_CLIPPED)  # the reference agrees


def _install_integration_stub(monkeypatch):
    """INTEGRATION.md §3 verbatim in substance: softmax_kit.gpu.softmax_gpu over
    the C ABI, and the `_USE_GPU` dispatch at the top of kernels.softmax."""
    errors, kernels, tensor = REF.errors, REF.kernels, REF.tensor
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    lib.sk_softmax_f32_host.restype = ctypes.c_int
    lib.sk_softmax_f32_host.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_int64)]
    lib.sk_last_error.restype = ctypes.c_char_p
    MODE = {kernels.KernelVariant.REFERENCE_CLIPPED: 0,
            kernels.KernelVariant.FULL_VECTORIZED_APPROX_EXP: 2}

    def softmax_gpu(m, variant, device=0):
        out = tensor.alloc_matrix(m.rows, m.cols)
        bad = ctypes.c_int64(-1)
        st = lib.sk_softmax_f32_host(m.data.ctypes.data, out.data.ctypes.data, m.rows, m.cols,
                                     MODE.get(variant, 1), device, ctypes.byref(bad))
        if st == 2:
            raise errors.NumericDomainError(f"non-finite logits in row {bad.value}")
        if st == 1:
            raise errors.ArgumentError(lib.sk_last_error().decode())
        if st == 4:
            raise errors.ResourceError(lib.sk_last_error().decode())
        if st != 0:
            raise errors.SoftmaxKitError(lib.sk_last_error().decode())
        return out

    gpu = types.ModuleType("softmax_kit.gpu")
    gpu.softmax_gpu = softmax_gpu
    monkeypatch.setitem(__import__("sys").modules, "softmax_kit.gpu", gpu)
    cpu_softmax = kernels.softmax

    def softmax(m, variant, cfg=REF.simd_reduce.LaneConfig()):
        return gpu.softmax_gpu(m, variant)  # `if _USE_GPU:` branch of INTEGRATION.md §3

    monkeypatch.setattr(kernels, "softmax", softmax)
    return cpu_softmax


@needs_ref
def test_integration_stub_inside_softmax_kit(monkeypatch, oracle):
    x = configs.generate("c3")
    m = _ref_matrix(x)
    V = REF.kernels.KernelVariant
    cpu_softmax = _install_integration_stub(monkeypatch)
    live = cpu_softmax(m, V.REFERENCE_CLIPPED)
    out = REF.kernels.softmax(m, V.REFERENCE_CLIPPED)   # the reference's entry point, now GPU
    assert type(out) is type(m)
    d = oracle.parity(out.view2d, live.view2d)
    assert d["ok"], d
    dev, _ = gu.softmax_abi(x)
    assert np.array_equal(out.view2d.view(np.uint32), dev.view(np.uint32))
    # every rung through the stub: unclipped rungs against the reference's Inference rung
    inf = cpu_softmax(m, V.REFERENCE_INFERENCE)
    for v in (V.REFERENCE_INFERENCE, V.MKL_STYLE_SCALAR, V.VECTORIZED_SUM, V.FULL_VECTORIZED):
        assert oracle.parity(REF.kernels.softmax(m, v).view2d, inf.view2d)["ok"], v
    ap = REF.kernels.softmax(m, V.FULL_VECTORIZED_APPROX_EXP)
    assert oracle.parity(ap.view2d, inf.view2d, approx=True)["ok"]
    bad = x.copy()
    bad[4000, 17] = np.inf
    with pytest.raises(REF.errors.NumericDomainError, match="row 4000"):
        REF.kernels.softmax(_ref_matrix(bad), V.REFERENCE_CLIPPED)
