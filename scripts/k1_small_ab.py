#!/usr/bin/env python
"""Short rows (C <= 64): the current default K1 plan vs the previous one
(forced through the K1 shape knobs), same buffers, at several job sizes; max
relative error against a float64 torch softmax (timing script check only)."""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "scripts"))

import torch  # noqa: E402

from paper_1904_12380_b200 import _native, configs  # noqa: E402
from sweep import bench_once  # noqa: E402


def old_shape(C):
    if C % 4 == 0:
        return (4, 1, 4, 0) if C <= 16 else (8, 1, 4, 0) if C <= 32 else (16, 1, 4, 0)
    return (8, 1, 4, 0) if C <= 8 else (16, 1, 4, 0) if C <= 16 else (32, 1, 4, 0) if C <= 32 \
        else (16, 4, 1, 1)


def main():
    cs = [8, 12, 16, 20, 24, 28, 32, 36, 40, 44, 48, 52, 56, 60, 64, 33, 45, 50, 57, 63]
    sizes = [16 << 20, 1 << 22, 1 << 21, 0]  # elements; 0 = 4096 rows
    s = torch.cuda.Stream()
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    for C in cs:
        for n in sizes:
            rows = n // C if n else 4096
            spec = configs.InputSpec(f"len{C}", rows, C, "normal", 7, sigma=4.0)
            x0 = torch.from_numpy(configs.generate(spec)).cuda()
            sh = (x0.double() - x0.double().amax(1, keepdim=True)).clamp_min(-64.0).exp_()
            ref = (sh / sh.sum(1, keepdim=True)).float()
            R = max(2, -(-3 * l2 // (8 * rows * C)))
            xs = [x0] + [x0.clone() for _ in range(R - 1)]
            ys = [torch.empty_like(x0) for _ in range(R)]
            rec = {"C": C, "rows": rows}
            for tag in ("new", "old"):
                if tag == "old":
                    lpr, nv, u, pf = old_shape(C)
                    for k, v in (("k1_lpr", lpr), ("k1_nv", nv), ("k1_u", u), ("k1_pf", pf),
                                 ("grid_mult", 0)):
                        _native.set_tuning(k, v)
                us = bench_once(xs, ys, rows, C, 100 if rows * C > (1 << 22) else 1000, s)
                torch.cuda.synchronize()
                rec[tag + "_us"] = round(us, 2)
                rec[tag + "_plan"] = _native.describe_plan(rows, C)
                rec[tag + "_max_rel"] = float(((ys[0] - ref).abs() / ref).max())
            for k, v in (("k1_lpr", 0), ("k1_nv", 0), ("k1_u", 0), ("k1_pf", -1), ("grid_mult", 0)):
                _native.set_tuning(k, v)
            rec["speedup"] = round(rec["old_us"] / rec["new_us"], 3)
            print(json.dumps(rec), flush=True)
            del xs, ys, x0, ref, sh


if __name__ == "__main__":
    main()
