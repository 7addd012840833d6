"""The page-locking cache for a caller's own pageable buffers (hostpin.py):
policy and lifetime on CPU with a recording stand-in for the C ABI; the real
registration and its effect on the host path on the GPU."""

import gc

import numpy as np
import pytest

import paper_1904_12380_b200 as sk
from paper_1904_12380_b200 import hostpin


class _FakeLib:
    def __init__(self, fail=False):
        self.reg, self.unreg, self.fail = [], [], fail

    def sk_host_register(self, ptr, nbytes):
        self.reg.append((ptr, nbytes))
        return 5 if self.fail else 0

    def sk_host_unregister(self, ptr):
        self.unreg.append(ptr)
        return 0


@pytest.fixture
def fake(monkeypatch):
    lib = _FakeLib()
    monkeypatch.setattr(hostpin._native, "lib", lambda: lib)
    before = hostpin.configure()
    hostpin.configure(enabled=True, min_bytes=1 << 10, sightings=2, budget_bytes=1 << 30)
    yield lib
    hostpin.release_all()
    hostpin.configure(enabled=before["enabled"], min_bytes=before["min_bytes"],
                      sightings=before["sightings"], budget_bytes=before["budget_bytes"])


def test_registers_on_second_sighting_and_releases_with_the_owner(fake):
    m = sk.alloc_matrix(64, 64)  # a view into an over-allocated np.zeros, like the reference's
    own = m.data.base
    assert not hostpin.note(m.view2d) and fake.reg == []
    assert hostpin.note(m.view2d)
    assert fake.reg == [(own.ctypes.data, own.nbytes)]
    assert hostpin.note(m.view2d[:40]) and len(fake.reg) == 1  # any view of the owner hits
    assert hostpin.stats()["bytes"] == own.nbytes
    ptr = own.ctypes.data
    del m, own
    gc.collect()
    assert fake.unreg == [ptr] and hostpin.stats() == {"ranges": 0, "bytes": 0, "tracked": 0}


def test_small_buffers_windows_and_disabled_are_left_alone(fake):
    small = np.zeros(16, np.float32)
    big = np.zeros(1 << 16, np.float32)
    for _ in range(3):
        assert not hostpin.note(small)
        assert not hostpin.note(big[:1024])  # a small window of a large owner
    hostpin.configure(enabled=False)
    for _ in range(3):
        assert not hostpin.note(big)
    assert fake.reg == []


def test_failed_registration_is_not_retried_and_budget_is_kept(fake):
    fake.fail = True
    a = np.zeros(4096, np.float32)
    assert not hostpin.note(a) and not hostpin.note(a) and not hostpin.note(a)
    assert len(fake.reg) == 1 and fake.unreg == []
    fake.fail = False
    hostpin.configure(budget_bytes=20000)
    b, c = np.zeros(4096, np.float32), np.zeros(4096, np.float32)
    hostpin.note(b), hostpin.note(c)
    assert hostpin.note(b) and not hostpin.note(c)  # 16 KiB fits the budget once
    del a, b, c
    gc.collect()
    assert hostpin.stats()["bytes"] == 0


def test_reused_address_is_a_new_buffer(fake):
    a = np.zeros(4096, np.float32)
    hostpin.note(a), hostpin.note(a)
    del a
    gc.collect()
    b = np.zeros(4096, np.float32)  # may land on the same address / id
    assert not hostpin.note(b)      # first sighting again
    assert len(fake.unreg) == 1


@pytest.mark.gpu
def test_pageable_matrix_is_pinned_on_second_call_same_bits():
    import torch

    from paper_1904_12380_b200 import configs

    before = hostpin.configure()
    hostpin.configure(enabled=True, min_bytes=1 << 20, sightings=2)
    try:
        x = configs.generate("c2")
        m = sk.Matrix2D.from_array(x)
        o = sk.alloc_matrix(*x.shape)
        ref = sk.softmax(torch.from_numpy(x).cuda(), sk.KernelVariant.REFERENCE_CLIPPED).cpu().numpy()
        base = hostpin.stats()["ranges"]
        sk.softmax(m, sk.KernelVariant.REFERENCE_CLIPPED, out=o)
        assert hostpin.stats()["ranges"] == base            # first call: staged
        assert np.array_equal(o.view2d.view(np.uint32), ref.view(np.uint32))
        o.view2d[:] = 0
        sk.softmax(m, sk.KernelVariant.REFERENCE_CLIPPED, out=o)
        assert hostpin.stats()["ranges"] == base + 2        # both buffers page-locked in place
        assert np.array_equal(o.view2d.view(np.uint32), ref.view(np.uint32))
        o.view2d[:] = 0
        sk.softmax(m, sk.KernelVariant.REFERENCE_CLIPPED, out=o)  # direct DMA path
        assert np.array_equal(o.view2d.view(np.uint32), ref.view(np.uint32))
        # a non-finite row is still reported with the right index on the direct path
        m.view2d[1234, 5] = np.inf
        with pytest.raises(sk.NumericDomainError, match="row 1234"):
            sk.softmax(m, sk.KernelVariant.REFERENCE_CLIPPED, out=o)
        del m, o
        gc.collect()
        assert hostpin.stats()["ranges"] == base            # released with the arrays
        # an already page-locked Matrix2D is never registered twice
        p = sk.Matrix2D.from_array(x, pinned=True)
        q = sk.alloc_matrix(*x.shape, pinned=True)
        for _ in range(3):
            sk.softmax(p, sk.KernelVariant.REFERENCE_CLIPPED, out=q)
        assert np.array_equal(q.view2d.view(np.uint32), ref.view(np.uint32))
        assert hostpin.stats()["ranges"] == base
    finally:
        hostpin.configure(enabled=before["enabled"], min_bytes=before["min_bytes"],
                          sightings=before["sightings"])
