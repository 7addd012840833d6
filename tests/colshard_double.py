"""Numpy test double for sharding.ColumnShardOps (CPU tests only).

It restates, in numpy, what the three native column-shard kernels compute
(include/softmax_b200.h: sk_row_stats_f32, sk_rescale_sumexp,
sk_normalize_f32) so the collective sequence in sharding.py can run on CPU
with a gloo process group.  It is a checker-side double, never a product path.
"""

from __future__ import annotations

import numpy as np
import torch

from paper_1904_12380_b200.sharding import ColumnShardOps

CLIP = np.float32(-64.0)
FLT_MIN = np.float32(np.finfo(np.float32).tiny)


def _exp_clip(x: np.ndarray, m: np.ndarray, clip: bool) -> np.ndarray:
    s = (x - m[:, None]).astype(np.float32)
    if clip:
        s = np.where(s > CLIP, s, CLIP).astype(np.float32)
    return np.exp(s.astype(np.float64)).astype(np.float32)


def numpy_column_ops() -> ColumnShardOps:
    def local_stats(x, mode):
        a = x.numpy()
        m = a.max(axis=1).astype(np.float32)
        s = _exp_clip(a, m, mode == 0).astype(np.float64).sum(axis=1)
        return torch.from_numpy(m), torch.from_numpy(s)

    def rescale(m_local, M, s):
        f = np.exp((m_local.numpy() - M.numpy()).astype(np.float32).astype(np.float64))
        return torch.from_numpy(s.numpy() * f.astype(np.float32).astype(np.float64))

    def normalize(x, M, S, mode):
        e = _exp_clip(x.numpy(), M.numpy(), mode == 0)
        r = (np.float32(1.0) / S.numpy().astype(np.float32)).astype(np.float32)
        y = (e * r[:, None]).astype(np.float32)
        y[y < FLT_MIN] = 0.0
        return torch.from_numpy(y)

    return ColumnShardOps(local_stats, rescale, normalize)
