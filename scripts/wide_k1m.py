#!/usr/bin/env python
"""Rows of 8193..16384 floats: K3g (grid-resident row; the default beyond
8192 until K1m took this range) vs K1m with a whole 256-thread block holding the row in registers
(`k1m_max_cols`), same buffers; max relative error against a float64 torch
softmax (timing script check only).  One JSON line per (shape, variant)."""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "scripts"))

import torch  # noqa: E402

from paper_1904_12380_b200 import _native, configs  # noqa: E402
from sweep import bench_once  # noqa: E402

SHAPES = [(1365, 12288), (4096, 12288), (16384, 12288), (1024, 16384), (4096, 16384),
          (16384, 16384), (2048, 10000), (8192, 10000), (2048, 12289), (4096, 16383),
          (8192, 9000)]


def main():
    shapes = SHAPES
    if len(sys.argv) > 1:  # RxC,...
        shapes = [tuple(map(int, t.split("x"))) for t in sys.argv[1].split(",")]
    s = torch.cuda.Stream()
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    for rows, cols in shapes:
        spec = configs.InputSpec(f"shape{rows}x{cols}", rows, cols, "normal", 11, sigma=4.0)
        x0 = torch.from_numpy(configs.generate(spec)).cuda()
        sh = (x0.double() - x0.double().amax(1, keepdim=True)).clamp_min(-64.0).exp_()
        ref = (sh / sh.sum(1, keepdim=True)).float()
        del sh
        R = max(2, -(-3 * l2 // (8 * rows * cols)))
        xs = [x0] + [x0.clone() for _ in range(R - 1)]
        ys = [torch.empty_like(x0) for _ in range(R)]
        for tag, kmax in (("k3g", 8192), ("k1m", 16384)):
            _native.set_tuning("k1m_max_cols", kmax)
            try:
                us = bench_once(xs, ys, rows, cols, 200, s)
                torch.cuda.synchronize()
                err = float(((ys[0] - ref).abs() / ref).max())
                print(json.dumps({"shape": [rows, cols], "variant": tag, "us": us,
                                  "gbs": 8.0 * rows * cols / us / 1e3, "max_rel": err,
                                  "plan": _native.describe_plan(rows, cols)}), flush=True)
            except Exception as e:  # noqa: BLE001
                print(json.dumps({"shape": [rows, cols], "variant": tag, "error": str(e)}), flush=True)
        _native.set_tuning("k1m_max_cols", 0)
        from row_length_sweep import copy_us  # noqa: E402

        cu = copy_us(xs, ys, rows * cols, 200, s)
        print(json.dumps({"shape": [rows, cols], "variant": "own copy", "us": cu,
                          "gbs": 8.0 * rows * cols / cu / 1e3}), flush=True)


if __name__ == "__main__":
    main()
