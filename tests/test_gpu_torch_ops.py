"""torch.ops.softmax_b200.* on the GPU: parity with the oracle, the column-shard
pieces composing to the full softmax, stream semantics and CUDA-graph capture."""

import numpy as np
import pytest
import torch

from paper_1904_12380_b200 import configs, torch_ops

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    return torch_ops.load()


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_softmax_fwd_parity(ops, name, oracle):
    x = configs.generate(name)
    xd = torch.from_numpy(x).cuda()
    for clip in (True, False):
        y = ops.softmax_fwd(xd, clip)
        assert y.shape == xd.shape and y.dtype == torch.float32
        d = oracle.parity(y.cpu().numpy(), oracle.softmax_ref(x, clip))
        assert d["ok"], (name, clip, d)


def test_softmax_fwd_out_long_rows_and_strided(ops, oracle):
    x = configs.generate("c4", 0, 5)
    big = torch.zeros(5, x.shape[1] + 64, device="cuda")
    big[:, :x.shape[1]] = torch.from_numpy(x).cuda()
    xs = big[:, :x.shape[1]]  # padded pitch
    y = torch.empty(5, x.shape[1], device="cuda")
    ops.softmax_fwd_out(xs, y, True)
    assert oracle.parity(y.cpu().numpy(), oracle.softmax_ref(x, True))["ok"]


def test_column_pieces_compose(ops, oracle):
    """row_max / row_sumexp / normalize_ over column shards == full softmax."""
    x = np.ascontiguousarray(configs.generate("c3")[:300])
    xd = torch.from_numpy(x).cuda()
    parts = [xd[:, a:b].contiguous() for a, b in ((0, 333), (333, 700), (700, 1000))]
    M = torch.stack([ops.row_max(p) for p in parts]).max(dim=0).values
    S = sum(ops.row_sumexp(p, M, True) for p in parts)
    outs = []
    for p in parts:
        y = torch.empty_like(p)
        ops.normalize_(p, M, S, y, True)
        outs.append(y)
    y = torch.cat(outs, dim=1).cpu().numpy()
    assert oracle.parity(y, oracle.softmax_ref(x, True))["ok"]


def test_errors_and_stream_and_graph(ops, oracle):
    with pytest.raises(RuntimeError, match="float32"):
        ops.softmax_fwd(torch.zeros(2, 3, device="cuda", dtype=torch.float64), True)
    with pytest.raises(RuntimeError, match="same shape"):
        ops.softmax_fwd_out(torch.zeros(2, 3, device="cuda"), torch.zeros(2, 4, device="cuda"),
                            True)
    x = configs.generate("c2", 0, 4096)
    xd = torch.from_numpy(x).cuda()
    y = torch.empty_like(xd)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ops.softmax_fwd_out(xd, y, True)  # warm-up (plans, workspace) outside capture
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            ops.softmax_fwd_out(xd, y, True)
    y.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert oracle.parity(y.cpu().numpy(), oracle.softmax_ref(x, True))["ok"]
