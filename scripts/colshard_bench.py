#!/usr/bin/env python
"""Per-rank cost of the column-sharded softmax (config c5b split n ways).

On one GPU: rank 0's [1024, C/n] shard runs the real kernels
(sk_row_stats_f32 -> rescale -> sk_normalize_f32); the two all-reduces are
replaced by device copies of the [N] vectors (the NCCL cost over NVLink is a
few-KiB latency term, reported separately by the multi-GPU run).  Prints one
JSON line per n with per-rank µs and effective GB/s (8 B/element of the shard).
"""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_1904_12380_b200 import configs, sharding  # noqa: E402


def main():
    spec = configs.get("c5b")
    ops = sharding.cuda_column_ops()
    for n in (1, 2, 4, 8):
        cols = spec.cols // n
        x = torch.empty(spec.rows, cols, device="cuda")
        x.normal_(0, 2.0, generator=torch.Generator("cuda").manual_seed(5))
        M = torch.empty(spec.rows, device="cuda")

        def step():
            m, s = ops.local_stats(x, 0)
            M.copy_(m)                       # all_reduce(MAX) stand-in
            s = ops.rescale(m, M, s)         # (no-op scale for one rank)
            return ops.normalize(x, M, s, 0)  # all_reduce(SUM) stand-in: identity

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record()
        for _ in range(reps):
            step()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / reps
        print(json.dumps({"n": n, "shard": [spec.rows, cols], "us_per_rank": us,
                          "gbs_per_rank": 8.0 * spec.rows * cols / us / 1e3,
                          "projected_aggregate_gbs": n * 8.0 * spec.rows * cols / us / 1e3}),
              flush=True)
        del x


if __name__ == "__main__":
    main()
