#!/usr/bin/env python
"""Column-sharded softmax (config c5b, [1024, 1048576]) split n ways, on one GPU.

Per world size n, one JSON line each for:

  split   rank 0's [1024, C/n] shard through the unfused path
          (sk_row_stats_f32 -> rescale -> sk_normalize_f32, 12 B/element); the
          two all-reduces are replaced by device copies of the [N] vectors.
  fused   rank 0's shard through the fused kernel (sk_colshard_softmax_f32,
          world = n) with gres_diag=1: the CTAs publish into all n exchange
          blocks but wait only for their own slot, so the number is the rank's
          streaming + in-kernel exchange cost WITHOUT the NVLink round trip
          (~1-2 us per row step, hidden behind the ring when lag >= 1) -- an
          estimate, labelled as such.
  emulate all n ranks of the full matrix as ONE cooperative kernel on this
          GPU (sk_colshard_emulate_f32): the real exchange between the
          virtual ranks; its time is the whole job on one GPU.

Effective GB/s = 8 B/element of the shard (or of the whole matrix for emulate).
"""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_1904_12380_b200 import _native, configs, sharding  # noqa: E402
from paper_1904_12380_b200.kernels import KernelVariant  # noqa: E402


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def main():
    spec = configs.get("c5b")
    ops = sharding.cuda_column_ops()
    nat = sharding.NativeExchange()
    blocks = [nat.alloc(0) for _ in range(8)]
    flag = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    xfull = torch.from_numpy(configs.generate(spec)).cuda()
    yfull = torch.empty_like(xfull)
    for n in (1, 2, 4, 8):
        cols = spec.cols // n
        x = xfull[:, :cols].contiguous()
        y = torch.empty_like(x)
        M = torch.empty(spec.rows, device="cuda")

        def split():
            m, s = ops.local_stats(x, 0)
            M.copy_(m)                       # all_reduce(MAX) stand-in
            s = ops.rescale(m, M, s)
            return ops.normalize(x, M, s, 0)  # all_reduce(SUM) stand-in: identity

        def fused():
            nat.launch(x, y, 0, 0, n, blocks[:n], flag)

        def emulate():
            sharding.emulate_column_shards(xfull, KernelVariant.REFERENCE_CLIPPED, n, out=yfull,
                                           check_finite=False)

        shard_bytes = 8.0 * spec.rows * cols
        us = timed(split, 10)
        print(json.dumps({"n": n, "path": "split", "shard": [spec.rows, cols], "us_per_rank": us,
                          "gbs_per_rank": shard_bytes / us / 1e3}), flush=True)
        _native.set_tuning("gres_diag", 1)
        try:
            us = timed(fused, 10)
        finally:
            _native.set_tuning("gres_diag", 0)
        print(json.dumps({"n": n, "path": "fused (own-slot wait: estimate)", "shard": [spec.rows, cols],
                          "plan": _native.describe_colshard_plan(spec.rows, cols, n),
                          "us_per_rank": us, "gbs_per_rank": shard_bytes / us / 1e3}), flush=True)
        us = timed(emulate, 5)
        print(json.dumps({"n": n, "path": "emulate (all ranks, one GPU)",
                          "plan": _native.describe_colshard_plan(spec.rows, cols, n, emulate=True),
                          "us_whole_job": us, "gbs": 8.0 * spec.rows * spec.cols / us / 1e3}),
              flush=True)
        del x, y
    assert int(flag.item()) == -1
    for b in blocks:
        nat.free(b)


if __name__ == "__main__":
    main()
