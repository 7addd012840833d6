"""GPU tests of the sharding layer on one B200.

Only one GPU is available per run, so n-way column sharding is emulated on
one device: each shard runs the real native kernels (sk_row_stats_f32 /
sk_rescale_sumexp / sk_normalize_f32); the all-reduce is replaced by the
equivalent torch max / sum over the shard statistics.  The real NCCL path
runs at world size 1.  (Multi-rank collectives are covered on CPU by
tests/test_sharding_gloo.py.)
"""

import os
import socket

import numpy as np
import pytest
import torch

import paper_1904_12380_b200 as sk
from paper_1904_12380_b200 import configs, sharding

pytestmark = pytest.mark.gpu


def _emulated_column_softmax(x, n, variant):
    ops = sharding.cuda_column_ops()
    mode = sk.variant_mode(variant)
    cols = x.shape[1]
    spans = [sharding.shard_range(cols, n, r) for r in range(n)]
    shards = [x[:, a:a + w].contiguous() for a, w in spans]
    stats = [ops.local_stats(s, mode) for s in shards]
    M = torch.stack([m for m, _ in stats]).max(dim=0).values          # all_reduce(MAX)
    S = sum(ops.rescale(m, M, s.clone()) for m, s in stats)           # all_reduce(SUM)
    return torch.cat([ops.normalize(s, M, S, mode) for s in shards], dim=1)


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_column_shards_emulated_c5b_rows(n, oracle):
    spec = configs.get("c5b")
    x = configs.generate(spec, 0, 6)
    xd = torch.from_numpy(x).cuda()
    y = _emulated_column_softmax(xd, n, sk.KernelVariant.REFERENCE_CLIPPED).cpu().numpy()
    d = oracle.parity(y, oracle.softmax_ref(x, True, nthreads=0))
    assert d["ok"], (n, d)


@pytest.mark.parametrize("n", [2, 3, 8])
def test_column_shards_emulated_clip_and_ragged(n, oracle):
    x = np.ascontiguousarray(configs.generate("c3")[:200, :997])
    xd = torch.from_numpy(x).cuda()
    for v in (sk.KernelVariant.REFERENCE_CLIPPED, sk.KernelVariant.REFERENCE_INFERENCE):
        y = _emulated_column_softmax(xd, n, v).cpu().numpy()
        ref = oracle.softmax_ref(x, v is sk.KernelVariant.REFERENCE_CLIPPED)
        assert oracle.parity(y, ref)["ok"], (n, v)


def test_nccl_world_size_one(oracle):
    import torch.distributed as dist

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        x = configs.generate("c5b", 0, 4)
        xd = torch.from_numpy(x).cuda()
        y = sharding.column_sharded_softmax(xd, sk.KernelVariant.REFERENCE_CLIPPED)
        assert oracle.parity(y.cpu().numpy(), oracle.softmax_ref(x, True, nthreads=0))["ok"]
        yr = sharding.row_sharded_softmax(xd, sk.KernelVariant.REFERENCE_CLIPPED)
        assert oracle.parity(yr.cpu().numpy(), oracle.softmax_ref(x, True, nthreads=0))["ok"]
    finally:
        dist.destroy_process_group()


def test_row_stats_device_matches_full_softmax(oracle):
    x = configs.generate("c4", 0, 3)
    st = sk.row_stats_device(torch.from_numpy(x).cuda())
    m = x.max(axis=1)
    assert np.array_equal(st.max.cpu().numpy(), m)
    s = np.exp(np.maximum(x - m[:, None], -64).astype(np.float64)).sum(axis=1)
    np.testing.assert_allclose(st.sum.cpu().numpy(), s, rtol=1e-6)
