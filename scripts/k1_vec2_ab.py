#!/usr/bin/env python
"""64-bit K1 rows (even row lengths on 8-B pitches, e.g. the paper's 50-word
attention rows) vs the 32-bit K1 plan they had before, plus forced 64-bit
shapes (LPR:NV:U): time per launch, this library's copy kernel of the same
bytes, max relative error against a float64 torch softmax.  One JSON line per
point."""

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


def reset():
    _native.set_tuning("vec2_max", 128)
    for k in ("k1_lpr", "k1_nv", "k1_u"):
        _native.set_tuning(k, 0)
    _native.set_tuning("k1_pf", -1)
    _native.set_tuning("k1_fit", 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cols", default="6,10,18,26,34,42,50,58,62,66,98,126,130,202,254")
    ap.add_argument("--mib", default="64,8")
    ap.add_argument("--rows4096", action="store_true", help="also 4096-row jobs (config c1's size)")
    ap.add_argument("--shapes", default="8:4:1,8:4:2,16:2:1,16:2:2,4:8:1,4:8:2,8:2:4,16:1:4,8:1:4",
                    help="forced 64-bit K1 shapes LPR:NV:U[:PF] (those covering C are run)")
    ap.add_argument("--vec1", action="store_true", help="forced shapes are 32-bit (odd rows)")
    ap.add_argument("--vw", type=int, default=2, help="vector width of the forced shapes (2, or 4 for 128-bit rows)")
    ap.add_argument("--ab", default="", help="A/B a tuning knob: <knob>[=<value>, default 0] against the default")
    ap.add_argument("--reps", type=int, default=2000)
    args = ap.parse_args()
    s = torch.cuda.Stream()
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    for C in map(int, args.cols.split(",")):
        sizes = [int(m) << 20 for m in args.mib.split(",")]
        row_counts = [sz // (4 * C) // 4 * 4 for sz in sizes] + ([4096] if args.rows4096 else [])
        for rows in row_counts:
            spec = configs.InputSpec(f"v{rows}x{C}", rows, C, "normal", 0, sigma=4.0)
            x0 = torch.from_numpy(configs.generate(spec)).cuda()
            R = max(2, -(-3 * l2 // (8 * rows * C)))
            xs = [x0] + [x0.clone() for _ in range(R - 1)]
            ys = [torch.empty_like(x0) for _ in range(R)]
            sh = (x0.double() - x0.double().amax(1, keepdim=True)).clamp_min(-64.0).exp_()
            ref = (sh / sh.sum(1, keepdim=True)).float()
            del sh
            cu = copy_us(xs, ys, rows * C, 50, s)
            if args.ab:
                knob, _, val = args.ab.partition("=")
                points = [(f"{knob}={val or 0}", {knob: int(val or 0)}), ("default", {})]
            else:
                points = [("v1", {"vec2_max": 0}), ("v2", {})]
            vw = 1 if args.vec1 else args.vw
            for shp in filter(None, args.shapes.split(",")):
                lpr, nv, u, pf = (list(map(int, shp.split(":"))) + [0])[:4]
                if C <= lpr * nv * vw < 2 * C:
                    t = {"k1_lpr": lpr, "k1_nv": nv, "k1_u": u, "k1_pf": pf}
                    if args.vec1:
                        t["vec2_max"] = 0
                    points.append((shp, t))
            for tag, tun in points:
                reset()
                for k, v in tun.items():
                    _native.set_tuning(k, v)
                rec = {"C": C, "rows": rows, "point": tag}
                try:
                    rec["plan"] = _native.describe_plan(rows, C)
                    us = bench_once(xs, ys, rows, C, args.reps, s)
                    torch.cuda.synchronize()
                    rec.update(us=round(us, 2), gbs=round(8.0 * rows * C / us / 1e3), copy_us=round(cu, 2),
                               vs_copy=round(cu / us, 3), max_rel=float(((ys[0] - ref).abs() / ref).max()))
                except Exception as e:  # noqa: BLE001
                    rec["error"] = str(e)[:100]
                print(json.dumps(rec), flush=True)
            reset()
            del xs, ys, x0, ref
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
