"""Page-locking cache for a drop-in caller's own host buffers.

The reference's ``alloc_matrix`` hands out pageable ``np.zeros`` memory
(tensor.py:90-103), and its timer calls ``softmax`` on the same two matrices
over and over (profiler.py:136-162).  From pageable memory every call pays two
host-side staging copies (sk_host.cu); from page-locked memory the DMA engines
read and write the caller's buffers directly (~95 vs ~53 GB/s on c5a).  Pinning
a buffer in place costs one to two staged calls (cudaHostRegister of 2 GiB:
35-50 ms when the range ends on a 2 MiB boundary, ~160 ms otherwise --
profiles/r2_hostreg_align.jsonl), so this cache does it only for a large buffer
seen for the SECOND time -- a one-shot call never pays it -- and releases the
registration when the owning ndarray dies (``weakref.finalize`` runs before
numpy frees the data), so no range stays registered past its memory.

The whole buffer of the owning ndarray is registered as ONE range: CUDA rejects
a copy whose host side spans two registrations (or leaves one), and the caller
-- or torch, for ``torch.from_numpy(a).cuda()`` -- may copy any part of its own
array at any time.  (Registering the inner 2 MiB-aligned window and the edge
pages separately is 4x faster and was tried: such a torch copy then fails with
"invalid argument".)  Only memory an ndarray OWNS is registered (never a window
onto someone else's buffer).  ``SK_HOST_PIN=0`` or ``configure(enabled=False)``
turns it off; the staged path is then always used for pageable memory.
"""

from __future__ import annotations

import mmap
import os
import threading
import weakref

import numpy as np

from . import _native

# re-entrant: dropping a pooled block (or any collection) under the lock can run
# an owner's finalizer (_release) on the same thread
_lock = threading.RLock()
_state = {
    "enabled": os.environ.get("SK_HOST_PIN", "1") != "0",
    "min_bytes": 512 << 10,       # below this the staging copy costs less than the bookkeeping
    "pool_min_bytes": 8 << 20,    # results at least this large come from the block pool
    "max_bytes": 64 << 30,        # never lock more than this in one range
    "sightings": 2,               # register on the N-th call that uses the buffer
    "budget_bytes": 0,            # 0: half of physical memory
}
_HUGE = 2 << 20
_entries: dict[int, "_Entry"] = {}
_pinned_total = 0


class _Entry:
    __slots__ = ("ptr", "nbytes", "seen", "box", "failed", "fin")

    def __init__(self, ptr: int, nbytes: int):
        self.ptr, self.nbytes = ptr, nbytes
        self.seen = 0
        self.box = [False]  # [registered]: shared with the owner's finalizer
        self.failed = False
        self.fin = None


def configure(enabled: bool | None = None, min_bytes: int | None = None,
              sightings: int | None = None, budget_bytes: int | None = None,
              pool_min_bytes: int | None = None) -> dict:
    """Set the cache policy; returns the policy in force."""
    with _lock:
        if enabled is not None:
            _state["enabled"] = bool(enabled)
        if min_bytes is not None:
            _state["min_bytes"] = int(min_bytes)
        if sightings is not None:
            _state["sightings"] = max(1, int(sightings))
        if budget_bytes is not None:
            _state["budget_bytes"] = max(0, int(budget_bytes))
        if pool_min_bytes is not None:
            _state["pool_min_bytes"] = max(0, int(pool_min_bytes))
        return dict(_state)


def stats() -> dict:
    with _lock:
        return {"ranges": sum(1 for e in _entries.values() if e.box[0]),
                "bytes": _pinned_total, "tracked": len(_entries)}


# ---------------------------------------------------- this package's own blocks
# Large matrices this package allocates itself (alloc_matrix, the result pool)
# are anonymous private mappings whose data window starts on a 2 MiB boundary
# and spans whole 2 MiB pages: transparent huge pages back it, cudaHostRegister
# of exactly that window takes 35-50 ms per 2 GiB instead of ~160 ms, and the
# DMA engines move page-aligned data (95 vs 85 GB/s).  Nothing outside the
# window is ever handed to anyone, so one registration of the window covers
# every copy a caller can make of the block's data.
_declared: dict[int, tuple[int, int]] = {}  # id(topmost ndarray) -> (window address, bytes)


def huge_block(nfloats: int) -> np.ndarray | None:
    """A zero-filled float32 buffer of ``nfloats`` whose first byte is on a
    2 MiB boundary, inside a private anonymous mapping of whole huge pages;
    None when the mapping cannot be made (the caller then uses numpy)."""
    win = (nfloats * 4 + _HUGE - 1) // _HUGE * _HUGE
    try:
        mm = mmap.mmap(-1, win + _HUGE, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS,
                       prot=mmap.PROT_READ | mmap.PROT_WRITE)
    except (OSError, ValueError, OverflowError):
        return None
    try:
        mm.madvise(mmap.MADV_HUGEPAGE)
    except (AttributeError, OSError, ValueError):
        pass
    raw = np.frombuffer(mm, dtype=np.uint8)
    off = (-raw.ctypes.data) % _HUGE
    key = id(raw)
    with _lock:
        _declared[key] = (raw.ctypes.data + off, win)
    weakref.finalize(raw, _declared.pop, key, None).atexit = False
    return raw[off: off + nfloats * 4].view(np.float32)


def _owner(a: np.ndarray) -> np.ndarray:
    while isinstance(a.base, np.ndarray):
        a = a.base
    return a


def _budget() -> int:
    b = _state["budget_bytes"]
    if b:
        return b
    try:
        return os.sysconf("SC_PHYS_PAGES") * os.sysconf("SC_PAGE_SIZE") // 2
    except (ValueError, OSError, AttributeError):
        return 16 << 30


def _release(key: int, ptr: int, nbytes: int, registered_box: list) -> None:
    """Finalizer of the owning ndarray: runs before numpy frees the data."""
    global _pinned_total
    with _lock:
        _entries.pop(key, None)
        if registered_box[0]:
            registered_box[0] = False
            _pinned_total -= nbytes
            try:
                _native.lib().sk_host_unregister(ptr)
            except Exception:  # noqa: BLE001 -- interpreter teardown
                pass


def note(view: np.ndarray) -> bool:
    """Record one host-path use of ``view``; page-lock its owner's buffer when
    the policy says so.  True when the buffer is registered after the call."""
    global _pinned_total
    if not _state["enabled"] or view.nbytes < _state["min_bytes"]:
        return False
    own = _owner(view)
    key = id(own)
    decl = _declared.get(key)
    if decl is not None and decl[0] <= view.ctypes.data and \
            view.ctypes.data + view.nbytes <= decl[0] + decl[1]:
        ptr, nbytes = decl  # one of this package's blocks: its aligned window
    else:
        ptr, nbytes = int(own.ctypes.data), int(own.nbytes)
        if not own.flags.owndata:
            # a window onto memory numpy does not own: its lifetime and its other
            # users are not ours to judge
            return False
    if nbytes > _state["max_bytes"] or view.nbytes * 2 < nbytes:
        return False  # a small part of a much larger buffer
    with _lock:
        e = _entries.get(key)
        if e is None or e.ptr != ptr or e.nbytes != nbytes:
            e = _Entry(ptr, nbytes)
            try:
                e.fin = weakref.finalize(own, _release, key, e.ptr, nbytes, e.box)
            except TypeError:
                return False
            e.fin.atexit = False  # process teardown releases every registration
            _entries[key] = e
        box = e.box
        if box[0]:
            return True
        if e.failed:
            return False
        e.seen += 1
        if e.seen < _state["sightings"] or _pinned_total + nbytes > _budget():
            return False
        if _native.lib().sk_host_register(e.ptr, nbytes) != 0:
            e.failed = True  # already registered by the caller, locked-memory limit, ...
            return False
        box[0] = True
        _pinned_total += nbytes
        return True


# ------------------------------------------------------------- output pool
# ``softmax(m, variant)`` returns a fresh Matrix2D per call (kernels.py:358).
# For a large result that means 2 GiB of first-touch page faults and a buffer
# the cache above never sees twice.  The pool keeps a few large output blocks
# alive and hands one out again once nothing but the pool references it (every
# view of a block -- the Matrix2D's data, its view2d, any slice the caller
# kept -- holds a reference to the block itself, so the block's reference
# count says exactly whether a caller can still see it).  A recycled block was
# seen before: note() page-locks it, and the call DMAs straight into it.
# Blocks are carved at a 2 MiB boundary, so the whole result is one aligned
# registration.  The result is fully overwritten by the call; it is NOT zeroed
# (alloc_matrix, which promises zeros, never uses the pool).
import sys  # noqa: E402

_POOL_MAX_BLOCKS = 4
_pool: list[tuple[np.ndarray, int]] = []  # (the block's topmost ndarray, floats handed out)


def _idle(i: int) -> bool:
    # references to the block's topmost array: the pool's tuple + getrefcount's
    # argument; every view handed out (and every view of a view) adds one
    return sys.getrefcount(_pool[i][0]) == 2


def pooled_output(nfloats: int) -> np.ndarray | None:
    """A float32 buffer of ``nfloats`` (2 MiB-aligned, uninitialised) from the
    pool, or None when the pool does not apply (small result, pool disabled or
    exhausted): the caller then allocates as usual."""
    nbytes = nfloats * 4
    if not _state["enabled"] or nbytes < max(_state["min_bytes"], _state["pool_min_bytes"]):
        return None
    with _lock:
        free = [i for i in range(len(_pool)) if _pool[i][1] == nfloats and _idle(i)]
        if free:
            top = _pool[free[0]][0]
            # a y = f(x) loop alternates between two blocks: keep one spare, let
            # the memory of any further idle block go
            for i in reversed(free[2:]):
                del _pool[i]
            lo = _declared[id(top)][0] - top.ctypes.data
            return top[lo: lo + nbytes].view(np.float32)
        # drop blocks of other sizes nobody uses; allocate while under the cap
        for i in range(len(_pool) - 1, -1, -1):
            if _pool[i][1] != nfloats and _idle(i):
                del _pool[i]
        held = sum(_declared[id(t)][1] for t, _ in _pool)
        if len(_pool) >= _POOL_MAX_BLOCKS or held + nbytes > _budget() // 2:
            return None
        data = huge_block(nfloats)
        if data is None:
            return None
        _pool.append((_owner(data), nfloats))
        return data


def pool_stats() -> dict:
    with _lock:
        return {"blocks": len(_pool), "bytes": sum(_declared[id(t)][1] for t, _ in _pool),
                "in_use": sum(1 for i in range(len(_pool)) if not _idle(i))}


def _after_fork_in_child() -> None:
    """A forked child has no CUDA context: its copies of the registrations are
    not its to release (the pages stay locked for the parent), so forget them
    rather than call the driver from the child when the arrays die."""
    global _pinned_total, _lock
    _lock = threading.RLock()
    for e in _entries.values():
        e.box[0] = False
        e.failed = True  # never try to lock the parent's buffers from the child
    _pinned_total = 0


if hasattr(os, "register_at_fork"):
    os.register_at_fork(after_in_child=_after_fork_in_child)


def release_all() -> None:
    """Drop every registration now (tests; a caller about to fork)."""
    with _lock:
        for i in range(len(_pool) - 1, -1, -1):
            if _idle(i):
                del _pool[i]
        fins = [e.fin for e in _entries.values() if e.fin is not None]
    for f in fins:
        f()
