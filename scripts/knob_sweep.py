#!/usr/bin/env python
"""Time arbitrary tuning-knob sets on arbitrary shapes, against this
library's copy kernel of the same bytes; max relative error against a
float64 torch softmax.  One JSON line per (shape, set).

    python scripts/knob_sweep.py --shapes 16384x1501,8192x3001 \\
        --sets "default;k1m_wpr=4,k1m_nv=12;path=2"
"""

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


# library defaults of the knobs a set may touch (sk_api.cu)
DEFAULTS = {"path": -1, "k1m_wpr": 0, "k1m_nv": 0, "k1_lpr": 0, "k1_nv": 0, "k1_u": 0, "k1_pf": -1,
            "gres": 1, "gres_p": 0, "gres_st": 0, "gres_lag": 0, "k3_impl": 3, "k1m": 1, "k1_fit": 1,
            "k1_wide32": 1280, "vec2_max": 128, "k4_fuse_combine": 1, "latency_steps": 3,
            "grid_mult": 0, "k1_threads": 128, "k1m_threads": 0}


def parse_sets(s):
    out = []
    for part in s.split(";"):
        part = part.strip()
        if not part or part == "default":
            out.append(("default", {}))
            continue
        kv = dict((k, int(v)) for k, v in (t.split("=") for t in part.split(",")))
        unknown = set(kv) - set(DEFAULTS)
        if unknown:
            raise SystemExit(f"no default recorded for {sorted(unknown)}")
        out.append((part, kv))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", required=True)
    ap.add_argument("--sets", default="default")
    ap.add_argument("--reps", type=int, default=300)
    args = ap.parse_args()
    s = torch.cuda.Stream()
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    sets = parse_sets(args.sets)
    for shp in args.shapes.split(","):
        rows, C = map(int, shp.split("x"))
        spec = configs.InputSpec(f"k{rows}x{C}", rows, C, "normal", 11, sigma=4.0)
        x0 = torch.from_numpy(configs.generate(spec)).cuda()
        R = max(2, -(-3 * l2 // (8 * rows * C)))
        xs = [x0] + [x0.clone() for _ in range(R - 1)]
        ys = [torch.empty_like(x0) for _ in range(R)]
        sh = (x0.double() - x0.double().amax(1, keepdim=True)).clamp_min(-64.0).exp_()
        ref = (sh / sh.sum(1, keepdim=True)).float()
        del sh
        n = rows * C
        cu = copy_us(xs, ys, n, 30, s) if n % 4 == 0 else None
        for tag, kv in sets:
            for k, v in kv.items():
                _native.set_tuning(k, v)
            rec = {"rows": rows, "cols": C, "set": tag}
            try:
                rec["plan"] = _native.describe_plan(rows, C)
                us = bench_once(xs, ys, rows, C, args.reps, s)
                torch.cuda.synchronize()
                rec.update(us=round(us, 2), gbs=round(8.0 * n / us / 1e3),
                           max_rel=float(((ys[0] - ref).abs() / ref).max()))
                if cu:
                    rec.update(copy_us=round(cu, 2), vs_copy=round(cu / us, 3))
            except Exception as e:  # noqa: BLE001
                rec["error"] = str(e)[:100]
            print(json.dumps(rec), flush=True)
            for k in kv:  # back to the library defaults
                _native.set_tuning(k, DEFAULTS[k])
        del xs, ys, x0, ref
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
