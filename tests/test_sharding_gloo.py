"""Multi-rank host logic of the sharding layer on CPU (gloo, world size 2/4).

Column sharding (config c5b's mode): each rank owns a column block; only the
per-row max (MAX) and sum (SUM) cross ranks.  The native kernels are replaced
by a numpy test double (tests/colshard_double.py); the collective sequence is
the product's sharding.column_sharded_softmax.  Row sharding needs no
collective: its ranges must tile the rows exactly.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1904_12380_b200 import sharding
from paper_1904_12380_b200.kernels import KernelVariant


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, x, variant_value, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from tests.colshard_double import numpy_column_ops

        c0, cn = sharding.shard_range(x.shape[1], world, rank)
        xl = torch.from_numpy(np.ascontiguousarray(x[:, c0:c0 + cn]))
        y = sharding.column_sharded_softmax(xl, KernelVariant(variant_value),
                                            ops=numpy_column_ops())
        out_q.put((rank, c0, y.numpy()))
    finally:
        dist.destroy_process_group()


def _run(world, x, variant):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, x, variant.value, q))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    parts.sort(key=lambda t: t[1])
    return np.concatenate([p[2] for p in parts], axis=1)


@pytest.mark.parametrize("world", [2, 4])
def test_column_sharded_softmax_gloo(world, oracle):
    from paper_1904_12380_b200 import configs

    x = configs.generate("c3")[:64]  # rows where the ValueClip fires
    x = np.ascontiguousarray(x[:, :999])  # ragged: 999 columns over `world` ranks
    y = _run(world, x, KernelVariant.REFERENCE_CLIPPED)
    ref = oracle.softmax_ref(x, True)
    d = oracle.parity(y, ref)
    assert d["ok"], d


def test_column_sharded_inference_mode_gloo(oracle):
    rng = np.random.default_rng(5)
    x = (rng.standard_normal((16, 257)) * 30).astype(np.float32)
    y = _run(2, x, KernelVariant.REFERENCE_INFERENCE)
    ref = oracle.softmax_ref(x, False)
    assert oracle.parity(y, ref)["ok"]


def test_shard_ranges_tile_exactly():
    for n in (0, 1, 7, 512, 2097152, 1048577):
        for world in (1, 2, 3, 4, 8):
            spans = [sharding.shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0
            for (a, na), (b, _) in zip(spans, spans[1:]):
                assert a + na == b
            assert spans[-1][0] + spans[-1][1] == n
            assert max(s[1] for s in spans) - min(s[1] for s in spans) <= 1
    with pytest.raises(Exception):
        sharding.shard_range(10, 2, 2)


def test_column_merge_math_matches_full_row(oracle):
    """(m_r, s_r) partials merged as max / rescaled sum equal the whole-row
    statistics, including when the clip fires in one shard only."""
    from tests.colshard_double import numpy_column_ops

    ops = numpy_column_ops()
    rng = np.random.default_rng(0)
    x = (rng.standard_normal((8, 600)) * 10).astype(np.float32)
    x[:, 5] = 300.0  # shard 0 holds the max -> other shards are far below it
    parts = np.split(x, [100, 350], axis=1)
    stats = [ops.local_stats(torch.from_numpy(np.ascontiguousarray(p)), 0) for p in parts]
    M = torch.stack([m for m, _ in stats]).max(dim=0).values
    S = sum(ops.rescale(m, M, s) for m, s in stats)
    y = np.concatenate([ops.normalize(torch.from_numpy(np.ascontiguousarray(p)), M, S, 0).numpy()
                        for p in parts], axis=1)
    assert oracle.parity(y, oracle.softmax_ref(x, True))["ok"]


class _FakeExchange:
    """Test double for sharding.NativeExchange: blocks are integers, handles
    name the block, "opening" a handle maps it to a distinct address."""

    MAP = 1 << 40

    def __init__(self):
        self.closed, self.freed, self.resets = [], [], []

    def alloc(self, device):
        return 0x1000 * (1 + int(os.environ["RANK"]))

    def handle(self, block):
        return f"blk:{block}".encode().ljust(64, b"\0")

    def open(self, handle):
        return self.MAP + int(handle.rstrip(b"\0").split(b":")[1])

    def close(self, block):
        self.closed.append(block)

    def free(self, block):
        self.freed.append(block)

    PERIOD = 3

    def reset_period(self):
        return self.PERIOD

    def reset(self, block):
        self.resets.append(block)


def _fused_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["RANK"] = str(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nat = _FakeExchange()
        fc = sharding.FusedColumnShard(device=0, native=nat)
        blocks = list(fc.blocks)
        fc.close()
        fc.close()  # idempotent
        out_q.put((rank, fc.world, fc.rank, blocks, nat.closed, nat.freed))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_fused_column_shard_handle_exchange_gloo(world):
    """Every rank maps every peer's exchange block (opened from the handle the
    peer published) and keeps its own at its rank index; close() unmaps the
    peers and frees its own block exactly once."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_fused_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, w, r, blocks, closed, freed in res:
        assert (w, r) == (world, rank)
        own = 0x1000 * (1 + rank)
        expect = [own if j == rank else _FakeExchange.MAP + 0x1000 * (1 + j) for j in range(world)]
        assert blocks == expect
        assert sorted(closed) == sorted(b for j, b in enumerate(expect) if j != rank)
        assert freed == [own]


def test_fused_column_shard_rejects_more_than_eight_ranks(monkeypatch):
    monkeypatch.setattr(dist, "is_initialized", lambda: True)
    monkeypatch.setattr(dist, "get_world_size", lambda group=None: 16)
    monkeypatch.setattr(dist, "get_rank", lambda group=None: 0)
    with pytest.raises(Exception, match="at most 8"):
        sharding.FusedColumnShard(device=0, native=_FakeExchange())


def _prepare_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["RANK"] = str(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nat = _FakeExchange()
        fc = sharding.FusedColumnShard(device=0, native=nat)
        log = []
        for call in range(8):
            before = len(nat.resets)
            fc._prepare(1024, 131072, 0)
            if len(nat.resets) > before:
                log.append(call)
        # a new shape on every rank, but rank 1's shard is wider: every rank refuses
        err = None
        try:
            fc._prepare(512, 131072 + (4 if rank == 1 else 0), 0)
        except Exception as e:  # noqa: BLE001
            err = type(e).__name__ + ": " + str(e)
        # a fresh instance whose very first call disagrees
        err2 = None
        fc2 = sharding.FusedColumnShard(device=0, native=_FakeExchange())
        try:
            fc2._prepare(1024, 131072, rank % 2)
        except Exception as e:  # noqa: BLE001
            err2 = type(e).__name__
        err = (err, err2)
        out_q.put((rank, log, nat.resets, err))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_fused_column_shard_reset_schedule_and_shape_agreement_gloo(world):
    """Host side of FusedColumnShard calls: (1) every
    reset_period() calls every rank zeroes its own exchange block between two
    barriers, at the same call index on all ranks (the 23-bit slot epoch never
    wraps); (2) a rank whose shard differs makes every rank raise instead of
    launching kernels that would poll mismatched slot layouts until the
    exchange timeout."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_prepare_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, log, resets, err in res:
        assert log == [3, 6], (rank, log)
        assert resets == [0x1000 * (1 + rank)] * 2
        assert err[0] is not None and err[0].startswith("ArgumentError"), err
        assert "differ across ranks" in err[0] and err[1] == "ArgumentError"
