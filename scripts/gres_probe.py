#!/usr/bin/env python
"""K3g diagnostics: time the grid-resident kernel with and without its group
exchange (gres_diag=1 skips it: results wrong, timing = the pipeline's own
bound) over a list of group sizes / ring depths.  One JSON line per point."""

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "scripts"))

import torch  # noqa: E402

from paper_1904_12380_b200 import _native, configs  # noqa: E402
from sweep import bench_once  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--points", default="14:3,16:3,20:4,24:4",
                    help="P:stages[:lag],... (lag 0 / absent: the classic lag for the depth)")
    ap.add_argument("--reps", type=int, default=60)
    ap.add_argument("--diags", default="0,1", help="gres_diag values: 1 skips the group exchange, 2 the math, 3 both")
    ap.add_argument("--sleeps", default="128", help="poller back-off values (ns)")
    ap.add_argument("--splits", default="-1", help="poller warp: -1 auto, 0 off, 1 on")
    args = ap.parse_args()
    spec = configs.get(args.config)
    x0 = torch.from_numpy(configs.generate(spec)).cuda()
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    R = max(2, -(-3 * l2 // (8 * spec.rows * spec.cols)))
    xs = [x0] + [x0.clone() for _ in range(R - 1)]
    ys = [torch.empty_like(x0) for _ in range(R)]
    s = torch.cuda.Stream()
    # float64 torch reference of the clipped softmax (timing script check only)
    sh = (x0.double() - x0.double().amax(1, keepdim=True)).clamp_min(-64.0).exp_()
    ref = (sh / sh.sum(1, keepdim=True)).float()
    del sh
    _native.set_tuning("gres", 2)
    for pt in args.points.split(","):
        P, st, lag = (list(map(int, pt.split(":"))) + [0])[:3]
        _native.set_tuning("gres_p", P)
        _native.set_tuning("gres_st", st)
        _native.set_tuning("gres_lag", lag)
        for d, sl, sp in [(d, sl, sp) for d in map(int, args.diags.split(","))
                          for sl in map(int, args.sleeps.split(","))
                          for sp in map(int, args.splits.split(","))]:
            _native.set_tuning("gres_diag", d)
            _native.set_tuning("gres_sleep", sl)
            _native.set_tuning("gres_split", sp)
            try:
                us = bench_once(xs, ys, spec.rows, spec.cols, args.reps, s)
            except Exception as e:  # noqa: BLE001
                print(json.dumps({"P": P, "stages": st, "lag": lag, "error": str(e)}), flush=True)
                continue
            rec = {"config": spec.name, "P": P, "stages": st, "lag": lag, "diag": d, "sleep": sl, "split": sp,
                   "us": us, "gbs": 8.0 * spec.rows * spec.cols / us / 1e3}
            if d == 0:
                torch.cuda.synchronize()
                y = ys[0]
                rec["max_rel"] = float(((y - ref).abs() / ref).max())
                rec["plan"] = _native.describe_plan(spec.rows, spec.cols)
            print(json.dumps(rec), flush=True)
    _native.set_tuning("gres_diag", 0)
    _native.set_tuning("gres_lag", 0)
    from row_length_sweep import copy_us  # noqa: E402

    cu = copy_us(xs, ys, spec.rows * spec.cols, args.reps, s)
    print(json.dumps({"config": spec.name, "copy_us": cu, "gbs": 8.0 * spec.rows * spec.cols / cu / 1e3}),
          flush=True)


if __name__ == "__main__":
    main()
