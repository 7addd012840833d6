#!/usr/bin/env python
"""Long-row shard sizes (c4 row-sharded n ways: 512/n rows x 262144; c5b
column-sharded: 1024 x 1M/n): the default plan against K3g (P, depth, lag)
points, K3g with parts switched off (gres_diag), K3c, the split path and this
library's copy kernel of the same bytes.  One JSON line per point."""

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "scripts"))

import torch  # noqa: E402

from paper_1904_12380_b200 import _native, configs  # noqa: E402
from row_length_sweep import copy_us  # noqa: E402
from sweep import bench_once  # noqa: E402

DEFAULTS = {"gres": 1, "gres_p": 0, "gres_st": 0, "gres_lag": 0, "gres_diag": 0, "path": -1, "k3_impl": 3,
            "k4_fuse_combine": 1, "latency_steps": 3}


def parse_points(s):
    out = [("default", {})]
    for tok in filter(None, s.split(",")):
        if tok == "k3c":
            out.append((tok, {"k3_impl": 5}))
        elif tok == "split":  # split path, row statistics merged inside normalize (2 launches)
            out.append((tok, {"path": 2}))
        elif tok == "split3":  # split path as three launches (stats, combine, normalize)
            out.append((tok, {"path": 2, "k4_fuse_combine": 0}))
        elif tok.startswith("lat"):  # lat<n>: latency path up to n K3g row steps per group
            out.append((tok, {"latency_steps": int(tok[3:])}))
        elif tok.startswith("t"):  # t<diag>: default plan with diag bits that keep results (experiments)
            out.append((tok, {"gres_diag": int(tok[1:])}))
        elif tok.startswith("d"):  # d<diag>: default plan, parts switched off
            out.append((tok, {"gres": 2, "gres_diag": int(tok[1:])}))
        else:  # P:st[:lag[:diag]]
            P, st, lag, dg = (list(map(int, tok.split(":"))) + [0, 0])[:4]
            out.append((tok, {"gres": 2, "gres_p": P, "gres_st": st, "gres_lag": lag, "gres_diag": dg}))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="64x262144,128x262144,256x262144,512x262144")
    ap.add_argument("--points", default="d1,d2,d3,14:3,16:3,18:3,12:2,21:4,29:5,37:6:2,split,k3c")
    ap.add_argument("--reps", type=int, default=400)
    args = ap.parse_args()
    s = torch.cuda.Stream()
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    for shp in args.shapes.split(","):
        rows, C = map(int, shp.split("x"))
        spec = configs.InputSpec(f"s{rows}x{C}", rows, C, "normal", 3, sigma=5.0)
        x0 = torch.from_numpy(configs.generate(spec)).cuda()
        R = max(2, -(-3 * l2 // (8 * rows * C)))
        xs = [x0] + [x0.clone() for _ in range(R - 1)]
        ys = [torch.empty_like(x0) for _ in range(R)]
        sh = (x0.double() - x0.double().amax(1, keepdim=True)).clamp_min(-64.0).exp_()
        ref = (sh / sh.sum(1, keepdim=True)).float()
        del sh
        cu = copy_us(xs, ys, rows * C, 50, s)
        for tag, tun in parse_points(args.points):
            for k, v in DEFAULTS.items():
                _native.set_tuning(k, v)
            for k, v in tun.items():
                _native.set_tuning(k, v)
            rec = {"rows": rows, "cols": C, "point": tag}
            try:
                rec["plan"] = _native.describe_plan(rows, C)[:60]
                us = bench_once(xs, ys, rows, C, args.reps, s)
                torch.cuda.synchronize()
                rec.update(us=round(us, 2), gbs=round(8.0 * rows * C / us / 1e3), copy_us=round(cu, 2),
                           vs_copy=round(cu / us, 3))
                if not tag.startswith("d"):
                    rec["max_rel"] = float(((ys[0] - ref).abs() / ref).max())
            except Exception as e:  # noqa: BLE001
                rec["error"] = str(e)[:100]
            print(json.dumps(rec), flush=True)
        for k, v in DEFAULTS.items():
            _native.set_tuning(k, v)
        del xs, ys, x0, ref
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
