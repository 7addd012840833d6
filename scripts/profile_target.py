#!/usr/bin/env python
"""Small, deterministic launch sequence for ncu / compute-sanitizer.

    python scripts/profile_target.py --config c4 --reps 3 [--rows N]

Runs `reps` softmax calls (default plan, ReferenceClipped) through the C ABI
on device-resident inputs and checks the last output against the oracle on a
few rows, so a profiled command is also a correct one.
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1904_12380_b200 import _native, configs  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c2")
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--rows", type=int, default=0, help="use only the first N rows")
    p.add_argument("--mode", type=int, default=0)
    p.add_argument("--shape", default="", help="RxC: synthetic N(0,4^2) matrix instead of a config")
    args = p.parse_args()
    import os

    for kv in os.environ.get("SK_TUNING", "").split():
        k, v = kv.split("=")
        _native.set_tuning(k, int(v))
    if args.shape:
        r, c = map(int, args.shape.lower().split("x"))
        spec = configs.InputSpec(f"shape{r}x{c}", r, c, "normal", 11, sigma=4.0)
    else:
        spec = configs.get(args.config)
    rows = args.rows or spec.rows
    x = configs.generate(spec)[:rows] if spec.plant_count else configs.generate(spec, 0, rows)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    flag = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    L = _native.lib()
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(args.reps):
        _native.check(L.sk_softmax_f32(xd.data_ptr(), yd.data_ptr(), rows, spec.cols, spec.cols,
                                       spec.cols, args.mode, flag.data_ptr(), None, 0, s))
    torch.cuda.synchronize()
    import oracle

    sel = np.unique(np.linspace(0, rows - 1, 4).astype(int))
    ref = oracle.softmax_ref(x[sel], clip=(args.mode == 0))
    d = oracle.parity(yd[torch.from_numpy(sel).cuda()].cpu().numpy(), ref, approx=args.mode == 2)
    print(args.config, _native.describe_plan(rows, spec.cols, spec.cols, spec.cols,
                                             xd.data_ptr(), yd.data_ptr(), 0), d)
    if not d["ok"] or int(flag.item()) != -1:
        sys.exit(1)


if __name__ == "__main__":
    main()
