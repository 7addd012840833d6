"""Drop-in type fidelity without a GPU: the reference's own KernelVariant,
LaneConfig and Matrix2D are accepted by this package's entry point, validated
like the reference validates them, and errors are catchable as the
reference's classes (VERDICT r1 missing #3)."""

import numpy as np
import pytest

import paper_1904_12380_b200 as sk
from paper_1904_12380_b200 import kernels
from tests import refpkg

REF = refpkg.load()
needs_ref = pytest.mark.skipif(REF is None, reason="baseline/_ref (softmax_kit) not installed")


@needs_ref
def test_reference_variants_map_by_value():
    for v in REF.kernels.KernelVariant:
        assert kernels.as_variant(v).value == v.value
        assert kernels.variant_mode(v) == kernels.variant_mode(kernels.as_variant(v))
    assert kernels.variant_mode(REF.kernels.KernelVariant.REFERENCE_CLIPPED) == 0


def test_foreign_non_variant_rejected():
    import enum

    class Other(enum.Enum):
        A = "NotAVariant"

    for bad in (Other.A, "ReferenceClipped", 3, None):
        with pytest.raises(sk.ArgumentError, match="expected a KernelVariant"):
            kernels.as_variant(bad)


@needs_ref
def test_reference_laneconfig_accepted():
    kernels._check_cfg(REF.simd_reduce.LaneConfig())
    kernels._check_cfg(REF.simd_reduce.LaneConfig(16))


@needs_ref
def test_reference_matrix_validated_and_errors_catchable_as_reference_classes():
    m = REF.tensor.alloc_matrix(4, 8)
    assert kernels._is_foreign_matrix(m)
    assert kernels._foreign_view(m, "input").shape == (4, 8)
    out = kernels._foreign_out(m)
    assert type(out) is type(m) and out.shape == m.shape and out.data.ctypes.data % 32 == 0
    # a broken foreign matrix (object.__setattr__ around the frozen dataclass)
    bad = REF.tensor.alloc_matrix(4, 8)
    object.__setattr__(bad, "data", np.zeros(32, np.float64))
    with pytest.raises(REF.errors.ArgumentError, match="expected float32"):
        sk.softmax(bad, REF.kernels.KernelVariant.REFERENCE_CLIPPED)
    with pytest.raises(sk.ArgumentError):
        sk.softmax(bad, REF.kernels.KernelVariant.REFERENCE_CLIPPED)
    e = kernels._foreign_error(m, sk.NumericDomainError("non-finite logits in row 3"))
    assert isinstance(e, REF.errors.NumericDomainError) and isinstance(e, sk.NumericDomainError)
    assert isinstance(e, ValueError) and str(e) == "non-finite logits in row 3"
