"""Multi-GPU sharding of the row softmax (one process per GPU, torchrun).

Row sharding (configs c4, c5a): rows are independent, so each rank runs the
single-GPU softmax on its contiguous row block -- no communication in the
data path.  The kernel plan depends only on C (and alignment, which a
contiguous row block preserves when C % 4 == 0), so a row computed on any
rank is bit-identical to the same row computed on one GPU.

Column sharding (config c5b): each rank holds the column block
[N, C_r] of every row.  Only per-row statistics cross NVLink:

    (m_r, s_r)  = local max and local sum of exp(clip(x - m_r))     (K4 stats)
    M           = all_reduce(m_r, MAX)                              (NCCL, N fp32)
    s_r        *= exp(m_r - M)                                      (rescale)
    S           = all_reduce(s_r, SUM)                              (NCCL, N fp64)
    y           = exp(clip(x - M)) * (1 / (float)S)                 (normalize)

This is the RowStats pair of the reference (kernels.py:108-112, 272-276)
merged the way context-parallel attention merges (m, l) partials.  The
collective sequence is expressed against a small ``ColumnShardOps`` interface
so the host logic can be exercised on CPU with gloo and a numpy test double
(tests/test_sharding_gloo.py); the product binds it to the CUDA kernels.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Any, Callable

from .errors import ArgumentError
from .kernels import KernelVariant, LaneConfig, softmax, variant_mode


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block of ``n`` items owned by ``rank``: (start, count).
    The first ``n % world`` ranks get one extra item."""
    if world < 1 or not 0 <= rank < world:
        raise ArgumentError(f"bad rank {rank} for world size {world}")
    if n < 0:
        raise ArgumentError("n must be >= 0")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def row_sharded_softmax(x_local, variant: KernelVariant, cfg: LaneConfig = LaneConfig(), **kw):
    """Softmax of this rank's row block: no collective (rows are independent)."""
    return softmax(x_local, variant, cfg, **kw)


@dataclass
class ColumnShardOps:
    """The three local kernels of the column-sharded softmax."""

    local_stats: Callable[[Any, int], tuple[Any, Any]]      # x -> (m f32[N], s f64[N])
    rescale: Callable[[Any, Any, Any], Any]                 # (m_local, M, s) -> s (in place ok)
    normalize: Callable[[Any, Any, Any, int], Any]          # (x, M, S, mode) -> y


def cuda_column_ops() -> ColumnShardOps:
    """Bind ColumnShardOps to the native kernels (sk_row_stats_f32,
    sk_rescale_sumexp, sk_normalize_f32)."""
    import torch

    from . import _native

    def stream_of(t):
        return torch.cuda.current_stream(t.device).cuda_stream

    def local_stats(x, mode):
        rows, cols = x.shape
        m = torch.empty(rows, dtype=torch.float32, device=x.device)
        s = torch.empty(rows, dtype=torch.float64, device=x.device)
        if rows:
            _native.check(_native.lib().sk_row_stats_f32(
                x.data_ptr(), rows, cols, x.stride(0) if rows > 1 else cols, mode, m.data_ptr(),
                s.data_ptr(), None, None, 0, stream_of(x)), "row_stats")
        return m, s

    def rescale(m_local, M, s):
        _native.check(_native.lib().sk_rescale_sumexp(
            m_local.data_ptr(), M.data_ptr(), s.data_ptr(), s.numel(), stream_of(s)), "rescale")
        return s

    def normalize(x, M, S, mode):
        rows, cols = x.shape
        y = torch.empty_like(x)
        if rows:
            ld = x.stride(0) if rows > 1 else cols
            _native.check(_native.lib().sk_normalize_f32(
                x.data_ptr(), y.data_ptr(), rows, cols, ld, cols, mode, M.data_ptr(),
                S.data_ptr(), stream_of(x)), "normalize")
        return y

    return ColumnShardOps(local_stats, rescale, normalize)


def column_sharded_softmax(x_local, variant: KernelVariant, group=None,
                           ops: ColumnShardOps | None = None, all_reduce=None):
    """Softmax over rows whose columns are split across the ranks of ``group``.

    ``x_local`` is this rank's [N, C_r] block; returns its [N, C_r] output.
    Two latency-bound all-reduces (N fp32 MAX, N fp64 SUM) are the only
    communication.  ``all_reduce(tensor, op_name)`` defaults to
    torch.distributed.all_reduce over ``group``.
    """
    mode = variant_mode(variant)
    if ops is None:
        ops = cuda_column_ops()
    if all_reduce is None:
        import torch.distributed as dist

        def all_reduce(t, op):
            dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM,
                            group=group)
            return t

    m_local, s = ops.local_stats(x_local, mode)
    M = all_reduce(_clone(m_local), "max")
    s = ops.rescale(m_local, M, s)
    S = all_reduce(s, "sum")
    return ops.normalize(x_local, M, S, mode)


def _clone(t):
    return t.clone() if hasattr(t, "clone") else t.copy()


# --------------------------------------------------------------------------
# Fused column shard: the collective inside the kernel
# --------------------------------------------------------------------------
class NativeExchange:
    """The exchange-block / IPC entry points of libsoftmax_b200 (C ABI)."""

    def __init__(self):
        from . import _native

        self._native = _native
        self.L = _native.lib()

    def alloc(self, device: int) -> int:
        import ctypes

        p = ctypes.c_void_p()
        self._native.check(self.L.sk_xchg_alloc(device, ctypes.byref(p)), "xchg_alloc")
        return int(p.value)

    def free(self, block: int) -> None:
        self._native.check(self.L.sk_xchg_free(block), "xchg_free")

    def reset_period(self) -> int:
        return int(self.L.sk_xchg_reset_period())

    def reset(self, block: int) -> None:
        """Zero the block on the current stream and wait for it."""
        import torch

        s = torch.cuda.current_stream()
        self._native.check(self.L.sk_xchg_reset(block, s.cuda_stream), "xchg_reset")
        s.synchronize()

    def handle(self, block: int) -> bytes:
        import ctypes

        buf = ctypes.create_string_buffer(self._native.SK_IPC_HANDLE_BYTES)
        self._native.check(self.L.sk_ipc_handle(block, buf), "ipc_handle")
        return buf.raw

    def open(self, handle: bytes) -> int:
        import ctypes

        p = ctypes.c_void_p()
        self._native.check(self.L.sk_ipc_open(handle, ctypes.byref(p)), "ipc_open")
        return int(p.value)

    def close(self, block: int) -> None:
        self._native.check(self.L.sk_ipc_close(block), "ipc_close")

    def launch(self, x, y, mode: int, rank: int, world: int, blocks: list[int], flag) -> None:
        import ctypes

        import torch

        rows, cols = x.shape
        arr = (ctypes.c_void_p * world)(*blocks)
        stream = torch.cuda.current_stream(x.device).cuda_stream
        self._native.check(self.L.sk_colshard_softmax_f32(
            x.data_ptr(), y.data_ptr(), rows, cols, x.stride(0) if rows > 1 else cols,
            y.stride(0) if rows > 1 else cols, mode, rank, world, arr, flag.data_ptr(), stream),
            "colshard_softmax")


class FusedColumnShard:
    """Column-sharded softmax as ONE kernel per rank.

    Each rank's K3g kernel (sk_gres.cuh) keeps its [N, C_r] row slices in
    shared memory and stores every CTA's per-row (max, sum) pair straight
    into all ranks' exchange blocks -- peer memory mapped over NVLink with
    cudaIpc -- then polls its own block and writes y.  The row-statistics
    all-reduce of ``column_sharded_softmax`` (two NCCL calls and 12 B/element
    of HBM traffic through the split kernels) becomes in-kernel stores
    overlapped with the streaming (8 B/element).

    Create once per (group, device) -- the exchange handles are swapped with
    one host all-gather -- then call for every softmax, in the same order on
    every rank.  ``native`` / ``all_gather`` are injectable so the host logic
    runs on CPU with gloo and a test double (tests/test_sharding_gloo.py).
    """

    def __init__(self, group=None, device: int | None = None, *, native=None, all_gather=None,
                 barrier=None):
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            self.world = dist.get_world_size(group)
            self.rank = dist.get_rank(group)
        else:
            self.world, self.rank = 1, 0
        if self.world > 8:
            raise ArgumentError("the fused column shard spans at most 8 GPUs (one NVLink domain)")
        if all_gather is None:
            def all_gather(obj):
                if self.world == 1:
                    return [obj]
                out = [None] * self.world
                dist.all_gather_object(out, obj, group=group)
                return out
        if barrier is None:
            def barrier():
                if self.world > 1:
                    dist.barrier(group=group)
        self._all_gather = all_gather
        self._barrier = barrier
        self._agreed = None  # the (rows, cols, mode) every rank last agreed on
        self._calls = 0
        if device is None:
            import torch

            device = torch.cuda.current_device()
        self.device = device
        self._n = native if native is not None else NativeExchange()
        self.block = self._n.alloc(device)
        handles = all_gather(self._n.handle(self.block))
        if len(handles) != self.world:
            raise ArgumentError("exchange handle all-gather returned the wrong count")
        self.blocks = [self.block if r == self.rank else self._n.open(h)
                       for r, h in enumerate(handles)]
        self._closed = False

    def __call__(self, x_local, variant: KernelVariant, out=None, check_finite: bool = True):
        import torch

        from .kernels import _bad_flag, _raise_if_aborted
        from .errors import NumericDomainError

        mode = variant_mode(variant)
        if self._closed:
            raise ArgumentError("FusedColumnShard is closed")
        if x_local.dim() != 2 or x_local.dtype != torch.float32 or not x_local.is_cuda:
            raise ArgumentError("x_local must be a CUDA float32 [N, C_r] tensor")
        rows, cols = x_local.shape
        if cols > 1 and x_local.stride(1) != 1:
            raise ArgumentError("x_local must have unit column stride")
        if out is None:
            y = torch.empty_like(x_local)
        else:
            if not isinstance(out, torch.Tensor) or not out.is_cuda or out.dtype != torch.float32:
                raise ArgumentError("out must be a CUDA float32 tensor")
            if tuple(out.shape) != (rows, cols) or out.device != x_local.device:
                raise ArgumentError(f"out must be [{rows}, {cols}] on {x_local.device}")
            if cols > 1 and out.stride(1) != 1:
                raise ArgumentError("out must have unit column stride")
            y = out
        self._prepare(rows, cols, mode, sync=torch.cuda.synchronize)
        flag = _bad_flag(torch, x_local.device)
        self._n.launch(x_local, y, mode, self.rank, self.world, self.blocks, flag)
        if check_finite:
            bad = int(flag.item())
            _raise_if_aborted(flag, bad)
            if bad != -1:
                flag.fill_(-1)
                raise NumericDomainError(f"non-finite logits in row {bad}")
        return y

    def _prepare(self, rows: int, cols: int, mode: int, sync=None) -> None:
        """Host side of one call, in the same order on every rank:

        * the first call, and every call whose (rows, shard width, mode)
          differs from this rank's previous call, all-gathers it and raises on
          every rank if any rank differs -- the K3g plan (slot layout, CTAs
          per row, ring depth) is a function of the shard width, so uneven
          shards would merge mismatched slots or poll until the exchange
          timeout.  (Calls, shape changes included, must be issued in the
          same order on every rank: a rank that changes shape alone waits in
          the all-gather instead of launching.);
        * every ``reset_period()`` calls all ranks quiesce and zero their
          own exchange block (the slot tags' 23-bit epoch then never wraps;
          sk_gres.cuh, gres_tag)."""
        key = (int(rows), int(cols), int(mode))
        if key != self._agreed:
            seen = [tuple(k) for k in self._all_gather(key)]
            if any(k != key for k in seen):
                raise ArgumentError(
                    "column shards differ across ranks (rows, shard width, mode): "
                    f"{seen}; every rank needs the same rows, the same number of columns and "
                    "the same variant")
            self._agreed = key
        period = max(1, int(self._n.reset_period()))
        if self._calls and self._calls % period == 0:
            if sync is not None:
                sync()
            self._barrier()  # no rank is still publishing into a peer's block
            self._n.reset(self.block)
            self._barrier()  # every block is zero before any rank launches again
        self._calls += 1

    def close(self) -> None:
        if self._closed:
            return
        for r, b in enumerate(self.blocks):
            if r != self.rank:
                self._n.close(b)
        self._n.free(self.block)
        self._closed = True

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


_emu_blocks: dict[tuple[int, int], list[int]] = {}


def emulate_column_shards(x, variant: KernelVariant, world: int, out=None, check_finite=True):
    """All ``world`` ranks of a column-sharded softmax of ``x`` [N, C] as ONE
    cooperative kernel on this GPU (shard r = columns [r*C/world, (r+1)*C/world)),
    with one exchange block per virtual rank -- the same kernel and exchange
    code as ``FusedColumnShard``, for testing with fewer GPUs than ranks."""
    import ctypes

    import torch

    from . import _native
    from .errors import NumericDomainError
    from .kernels import _bad_flag, _raise_if_aborted

    mode = variant_mode(variant)
    rows, cols = x.shape
    dev = x.device.index if x.device.index is not None else torch.cuda.current_device()
    key = (dev, world)
    if key not in _emu_blocks:
        nat = NativeExchange()
        _emu_blocks[key] = [nat.alloc(dev) for _ in range(world)]
    blocks = _emu_blocks[key]
    y = torch.empty_like(x) if out is None else out
    flag = _bad_flag(torch, x.device)
    arr = (ctypes.c_void_p * world)(*blocks)
    _native.check(_native.lib().sk_colshard_emulate_f32(
        x.data_ptr(), y.data_ptr(), rows, cols, x.stride(0) if rows > 1 else cols,
        y.stride(0) if rows > 1 else cols, mode, world, arr, flag.data_ptr(),
        torch.cuda.current_stream(x.device).cuda_stream), "colshard_emulate")
    if check_finite:
        bad = int(flag.item())
        _raise_if_aborted(flag, bad)
        if bad != -1:
            flag.fill_(-1)
            raise NumericDomainError(f"non-finite logits in row {bad}")
    return y
