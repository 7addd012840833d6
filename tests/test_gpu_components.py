"""The 1-D component operations (kernels.py:229-276) on the GPU
(paper_1904_12380_b200.components) against the reference's own outputs
(tests/golden/golden_components.npz, made by make_golden_components.py)."""

import numpy as np
import pytest
import torch

import paper_1904_12380_b200 as sk
from paper_1904_12380_b200 import components as C

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def rows(g):
    return sorted({k.split("/")[0] for k in g.files if k.endswith("/row")})


def test_components_match_reference(golden_components):
    g = golden_components
    for name in rows(g):
        r = g[f"{name}/row"]
        m = C.row_max_scalar(r)
        assert isinstance(m, np.float32) and bits(m) == bits(g[f"{name}/max"][0]), name
        # exact IEEE elementwise ops: bit-identical
        assert np.array_equal(bits(C.subtract_broadcast(r, m)), bits(g[f"{name}/sub_max"])), name
        assert np.array_equal(bits(C.subtract_broadcast(r, 3.25)), bits(g[f"{name}/sub_325"])), name
        e_ref = g[f"{name}/exp"]
        assert np.array_equal(bits(C.scale_reciprocal(e_ref, g[f"{name}/sum_exp"][0])),
                              bits(g[f"{name}/scaled"])), name
        # exp: this library's exponential (<= 2.53 ulp) vs numpy's; subnormal
        # results (below FLT_MIN) to within a few units of 2^-149
        e = C.exp_batch(g[f"{name}/sub_max"].copy())
        np.testing.assert_allclose(e, e_ref, rtol=8e-7, atol=4 * 2.0 ** -149, err_msg=name)
        # f64 accumulation in another order, rounded to f32: equal, or 1 ulp at a tie
        for got, want in ((C.row_sum_scalar(e_ref), g[f"{name}/sum_exp"][0]),
                          (C.row_sum_scalar(r), g[f"{name}/sum_row"][0])):
            d = int(bits(got).reshape(-1)[0]) - int(bits(want).reshape(-1)[0])
            assert abs(d) <= 1, (name, got, want)
        st = C.row_stats(r)
        assert bits(st.max) == bits(g[f"{name}/stats"][0]), name
        np.testing.assert_allclose(st.sum, g[f"{name}/stats"][1], rtol=1e-6, err_msg=name)
    for x, y in zip(g["clip/x"], g["clip/y"]):
        assert bits(C.value_clip(x)) == bits(y)


def test_components_on_device_tensors(golden_components):
    g = golden_components
    r = g["u1000/row"]
    d = torch.from_numpy(r).cuda()
    m = C.row_max_scalar(d)
    assert m.is_cuda and float(m) == float(g["u1000/max"][0])
    sh = C.subtract_broadcast(d, float(m))
    assert sh.is_cuda and np.array_equal(bits(sh.cpu().numpy()), bits(g["u1000/sub_max"]))
    e = C.exp_batch(sh)  # in place
    assert e.data_ptr() == sh.data_ptr()
    s = C.row_sum_scalar(e)
    y = C.scale_reciprocal(e, float(s))
    np.testing.assert_allclose(y.cpu().numpy(), g["u1000/scaled"], rtol=1e-6)
    st = C.row_stats(d)
    assert st.max.is_cuda and float(st.max) == float(g["u1000/stats"][0])
    # the components compose into the fused kernel's answer (unclipped rung)
    full = sk.softmax(d.view(1, -1), sk.KernelVariant.REFERENCE_INFERENCE)
    np.testing.assert_allclose(y.cpu().numpy(), full.cpu().numpy()[0], rtol=2e-6, atol=1e-12)


def test_component_argument_errors():
    with pytest.raises(sk.ArgumentError):
        C.row_max_scalar(np.zeros((2, 3), np.float32))
    with pytest.raises(sk.ArgumentError):
        C.row_sum_scalar(np.zeros(0, np.float32))
    with pytest.raises(sk.ArgumentError):
        C.exp_batch(np.zeros(4, np.float64))
    with pytest.raises(sk.NumericDomainError):
        C.scale_reciprocal(np.ones(3, np.float32), 0.0)
    with pytest.raises(sk.NumericDomainError):
        C.scale_reciprocal(np.ones(3, np.float32), float("inf"))
    with pytest.raises(sk.ArgumentError):
        C.subtract_broadcast(torch.zeros(3), 1.0)  # CPU tensor: no CPU path
