"""The page-locking cache for a caller's own pageable buffers (hostpin.py):
policy and lifetime on CPU with a recording stand-in for the C ABI; the real
registration and its effect on the host path on the GPU."""

import gc

import numpy as np
import pytest

import paper_1904_12380_b200 as sk
from paper_1904_12380_b200 import hostpin


_M2 = 2 << 20


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
    hostpin.configure(enabled=True, min_bytes=1 << 20, sightings=2, budget_bytes=1 << 30,
                      pool_min_bytes=1 << 20)
    yield lib
    hostpin.release_all()
    hostpin.configure(enabled=before["enabled"], min_bytes=before["min_bytes"],
                      sightings=before["sightings"], budget_bytes=before["budget_bytes"],
                      pool_min_bytes=before["pool_min_bytes"])


def test_registers_on_second_sighting_and_releases_with_the_owner(fake):
    raw = np.zeros(4 * 1024 * 1024 + 8, np.float32)  # the reference allocator's layout
    off = (-raw.ctypes.data) % 32 // 4
    m = sk.Matrix2D(rows=2048, cols=2048, data=raw[off:off + 4 * 1024 * 1024])
    assert not hostpin.note(m.view2d) and fake.reg == []
    assert hostpin.note(m.view2d)
    # the owner's whole buffer as ONE range: a copy of any part of the caller's
    # array (torch.from_numpy(a).cuda()) must never straddle a registration
    assert fake.reg == [(raw.ctypes.data, raw.nbytes)]
    assert hostpin.note(m.view2d[:1200]) and len(fake.reg) == 1  # any view of the owner hits
    assert hostpin.stats()["bytes"] == raw.nbytes
    ptr = raw.ctypes.data
    del m, raw
    gc.collect()
    assert fake.unreg == [ptr] and hostpin.stats() == {"ranges": 0, "bytes": 0, "tracked": 0}


def test_this_packages_matrices_are_aligned_windows_of_whole_huge_pages(fake):
    m = sk.alloc_matrix(2048, 2049)                  # 16 MiB + 8 KiB: zero-filled, 2 MiB-aligned
    assert m.data.ctypes.data % _M2 == 0 and not m.data.any() and m.data.flags.writeable
    m.view2d[5, 7] = 3.0
    assert float(m.data[5 * 2049 + 7]) == 3.0
    hostpin.note(m.view2d), hostpin.note(m.view2d)
    win = (m.data.nbytes + _M2 - 1) // _M2 * _M2
    assert fake.reg == [(m.data.ctypes.data, win)]   # exactly the window, nothing outside it
    assert hostpin.note(m.view2d[100:1900])
    ptr = m.data.ctypes.data
    del m
    gc.collect()
    assert fake.unreg == [ptr] and hostpin.stats()["tracked"] == 0
    small = sk.alloc_matrix(64, 64)                  # small matrices stay plain numpy
    assert small.data.base.flags.owndata and small.data.ctypes.data % 32 == 0


def test_memory_numpy_does_not_own_is_never_registered(fake):
    backing = bytearray(8 << 20)
    a = np.frombuffer(backing, dtype=np.float32)
    for _ in range(3):
        assert not hostpin.note(a)
    assert fake.reg == []


def test_small_buffers_windows_and_disabled_are_left_alone(fake):
    small = np.zeros(1 << 10, np.float32)
    big = np.zeros(8 << 20, np.float32)
    for _ in range(3):
        assert not hostpin.note(small)
        assert not hostpin.note(big[: 1 << 20])  # a small window of a large owner
    hostpin.configure(enabled=False)
    for _ in range(3):
        assert not hostpin.note(big)
    assert fake.reg == []


def test_failed_registration_is_not_retried_and_budget_is_kept(fake):
    fake.fail = True
    a = np.zeros(2 << 20, np.float32)
    assert not hostpin.note(a) and not hostpin.note(a) and not hostpin.note(a)
    assert len(fake.reg) == 1 and fake.unreg == []
    fake.fail = False
    hostpin.configure(budget_bytes=10 << 20)
    b, c = np.zeros(2 << 20, np.float32), np.zeros(2 << 20, np.float32)
    hostpin.note(b), hostpin.note(c)
    assert hostpin.note(b) and not hostpin.note(c)  # 8 MiB fits the budget once
    del a, b, c
    gc.collect()
    assert hostpin.stats()["bytes"] == 0


def test_forked_child_forgets_the_parents_registrations(fake):
    import os

    a = np.zeros(2 << 20, np.float32)
    hostpin.note(a), hostpin.note(a)
    assert hostpin.stats()["ranges"] == 1
    r, w = os.pipe()
    pid = os.fork()
    if pid == 0:  # child: no CUDA context of its own
        try:
            ok = hostpin.stats()["ranges"] == 0 and not hostpin.note(a)
            del a
            gc.collect()
            ok = ok and fake.unreg == []  # the child never calls the driver for them
            os.write(w, b"1" if ok else b"0")
        finally:
            os._exit(0)
    os.close(w)
    assert os.read(r, 1) == b"1"
    os.waitpid(pid, 0)
    assert hostpin.stats()["ranges"] == 1  # the parent's registration is untouched


def test_reused_address_is_a_new_buffer(fake):
    a = np.zeros(2 << 20, np.float32)
    hostpin.note(a), hostpin.note(a)
    del a
    gc.collect()
    b = np.zeros(2 << 20, np.float32)  # may land on the same address / id
    assert not hostpin.note(b)      # first sighting again
    assert len(fake.unreg) == 1


@pytest.mark.timeout(60)
def test_output_pool_recycles_only_blocks_nobody_can_see(fake):
    n = 1 << 20  # 4 MiB results
    assert hostpin.pooled_output(1 << 10) is None              # small: not pooled
    a = hostpin.pooled_output(n)
    assert a.size == n and a.ctypes.data % (2 << 20) == 0 and a.dtype == np.float32
    b = hostpin.pooled_output(n)
    assert b.base is not a.base and hostpin.pool_stats()["in_use"] == 2
    a[:] = 7.0
    keep = a.reshape(1024, 1024)[5]                             # a slice the caller kept
    block = a.base
    del a
    c = hostpin.pooled_output(n)
    assert c.base is not block and float(keep[0]) == 7.0        # still visible: not reused
    del keep, block
    d = hostpin.pooled_output(n)
    assert d.base is not b.base and d.base is not c.base        # the released block comes back
    assert hostpin.pool_stats()["blocks"] == 3
    e = hostpin.pooled_output(n)
    assert e is not None and hostpin.pool_stats()["blocks"] == 4
    assert hostpin.pooled_output(n) is None                     # pool exhausted: caller allocates
    hostpin.note(e), hostpin.note(e)                            # registered: has a finalizer
    assert len(fake.reg) == 1
    del b, c, d, e
    assert hostpin.pool_stats()["in_use"] == 0
    g = hostpin.pooled_output(n)                                # 4 idle blocks: one handed out,
    assert hostpin.pool_stats()["blocks"] == 2                  # one spare kept, two released
    del g
    f = hostpin.pooled_output(2 * n)                            # another size evicts idle blocks
    assert len(fake.unreg) == 1                                 # ... releasing them (no deadlock)
    assert f is not None and hostpin.pool_stats()["blocks"] == 1
    hostpin.configure(enabled=False)
    assert hostpin.pooled_output(n) is None
    del f
    hostpin.release_all()
    assert hostpin.pool_stats()["blocks"] == 0


@pytest.mark.gpu
def test_fresh_outputs_come_from_the_pool_and_stay_valid():
    import torch

    from paper_1904_12380_b200 import configs

    before = hostpin.configure()
    hostpin.configure(enabled=True, min_bytes=1 << 20, sightings=2, pool_min_bytes=1 << 20)
    try:
        x = configs.generate("c2")
        ref = sk.softmax(torch.from_numpy(x).cuda(), sk.KernelVariant.REFERENCE_CLIPPED).cpu().numpy()
        m = sk.Matrix2D.from_array(x)
        outs = [sk.softmax(m, sk.KernelVariant.REFERENCE_CLIPPED) for _ in range(3)]  # all alive
        assert len({o.data.base.ctypes.data for o in outs}) == 3
        y = None
        for _ in range(6):                                       # the usual loop: y rebound
            y = sk.softmax(m, sk.KernelVariant.REFERENCE_CLIPPED)
            assert np.array_equal(y.view2d.view(np.uint32), ref.view(np.uint32))
        for o in outs:                                           # never overwritten meanwhile
            assert np.array_equal(o.view2d.view(np.uint32), ref.view(np.uint32))
        assert hostpin.pool_stats()["blocks"] <= 4
        assert hostpin.stats()["ranges"] >= 2                    # input + a recycled block
        # the reference's own Matrix2D class gets pooled outputs too (duck-typed path)
        x2 = x.copy()
        x2[7, 3] = np.nan
        with pytest.raises(sk.NumericDomainError, match="row 7"):
            sk.softmax(sk.Matrix2D.from_array(x2), sk.KernelVariant.REFERENCE_CLIPPED)
    finally:
        del outs, y, m
        gc.collect()
        hostpin.release_all()
        hostpin.configure(enabled=before["enabled"], min_bytes=before["min_bytes"],
                          sightings=before["sightings"], pool_min_bytes=before["pool_min_bytes"])


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


@pytest.mark.gpu
def test_host_path_fuzz_pinned_views_and_edges():
    """Random shapes / views through the host path while buffers move from
    staged to page-locked (whole owner, sub-views, odd byte offsets inside the
    registered window and across its edges): always the device path's bits."""
    import torch

    before = hostpin.configure()
    hostpin.configure(enabled=True, min_bytes=1 << 20, sightings=2)
    rng = np.random.default_rng(20260710)
    try:
        for case in range(24):
            cols = int(rng.choice([50, 128, 256, 1000, 1501, 4096, 20000, 70001]))
            rows = max(2, int((rng.integers(3, 40) << 20) // (4 * cols)))
            lead = int(rng.integers(0, 3)) * int(rng.choice([1, 8, 1024, 524288]))  # floats before the data
            raw_x = np.zeros(rows * cols + lead + 16, np.float32)
            raw_y = np.zeros(rows * cols + lead + 16, np.float32)
            x = raw_x[lead:lead + rows * cols].reshape(rows, cols)
            y = raw_y[lead:lead + rows * cols].reshape(rows, cols)
            x[:] = rng.standard_normal((rows, cols), dtype=np.float32) * 4
            ref = sk.softmax(torch.from_numpy(x).cuda(), sk.KernelVariant.REFERENCE_CLIPPED).cpu().numpy()
            # Long rows: a small standalone device call takes the latency path
            # (split) where the host path's chunks keep the throughput plan (K3g),
            # and K3g's unaligned variant cuts slices at each row's 16-B phase,
            # which differs between a chunk in a staging slot and the whole matrix
            # on the device (DESIGN sections 4-5): same values within the gate
            # there, the same bits for every row one CTA holds (<= 16384 floats)
            exact = cols <= 16384

            def same(a, b):
                if exact:
                    return np.array_equal(a.view(np.uint32), b.view(np.uint32))
                return bool((np.abs(a - b) <= 1e-5 * b).all())

            first = None
            for call in range(3):                      # staged, pinning, direct
                y[:] = -1.0
                out = sk.softmax(x, sk.KernelVariant.REFERENCE_CLIPPED, out=y)
                assert out is y
                assert same(y, ref), (case, call, rows, cols, lead)
                if first is None:
                    first = y.copy()
                # staged or direct, the host path itself always gives the same bits
                assert np.array_equal(y.view(np.uint32), first.view(np.uint32)), (case, call)
            # other CUDA users of the caller's memory keep working on the page-locked
            # buffer: any part of it, the whole owner included, copies in one piece
            assert torch.equal(torch.from_numpy(raw_y).cuda().cpu(), torch.from_numpy(raw_y))
            # a row block of the (now page-locked) buffers: same bits as those rows of the whole
            r0, r1 = sorted(int(v) for v in rng.integers(0, rows + 1, 2))
            if r1 - r0 >= 1:
                y[:] = -1.0
                sk.softmax(x[r0:r1], sk.KernelVariant.REFERENCE_CLIPPED, out=y[r0:r1])
                got = sk.softmax(torch.from_numpy(x[r0:r1]).cuda(),
                                 sk.KernelVariant.REFERENCE_CLIPPED).cpu().numpy()
                assert same(y[r0:r1], got), (case, r0, r1)
                assert (y[:r0] == -1.0).all() and (y[r1:] == -1.0).all()
            del x, y, raw_x, raw_y, out
            gc.collect()
        assert hostpin.stats()["bytes"] == 0
    finally:
        hostpin.release_all()
        hostpin.configure(enabled=before["enabled"], min_bytes=before["min_bytes"],
                          sightings=before["sightings"])
