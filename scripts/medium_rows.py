#!/usr/bin/env python
"""Medium rows (1024 < C <= 8192): K2 (TMA block-per-row, default) vs K1 with a
whole warp holding the row in registers (NV float4 per lane), same buffers."""

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
    shapes = [(65536, 1536, 16), (32768, 2048, 16), (16384, 3072, 24), (16384, 4096, 32),
              (4096, 4000, 32)]
    if len(sys.argv) > 1:  # RxCxNV,...
        shapes = [tuple(map(int, t.split("x"))) for t in sys.argv[1].split(",")]
    for rows, cols, nv in shapes:
        spec = configs.InputSpec(f"shape{rows}x{cols}", rows, cols, "normal", 11, sigma=4.0)
        x0 = torch.from_numpy(configs.generate(spec)).cuda()
        l2 = torch.cuda.get_device_properties(0).L2_cache_size
        R = max(2, -(-3 * l2 // (8 * rows * cols)))
        xs = [x0] + [x0.clone() for _ in range(R - 1)]
        ys = [torch.empty_like(x0) for _ in range(R)]
        s = torch.cuda.Stream()
        variants = [("default", {})]
        if cols <= 3072:
            for gm in (0, 2):
                variants.append((f"k1 lpr=32 nv={nv} gm={gm}",
                                 {"path": 0, "k1_lpr": 32, "k1_nv": nv, "k1_u": 1, "grid_mult": gm}))
        else:
            variants.append(("k2 (k1m off)", {"k1m": 0}))
            for wpr, nv2 in ((2, 16), (4, 8), (4, 12), (4, 16), (8, 8)):
                if wpr * 32 * nv2 * 4 >= cols:
                    variants.append((f"k1m wpr={wpr} nv={nv2}",
                                     {"path": 3, "k1m_wpr": wpr, "k1m_nv": nv2}))
        for tag, tun in variants:
            for k, v in tun.items():
                _native.set_tuning(k, v)
            try:
                us = bench_once(xs, ys, rows, cols, 200, s)
                print(json.dumps({"shape": [rows, cols], "variant": tag, "us": us,
                                  "gbs": 8.0 * rows * cols / us / 1e3,
                                  "plan": _native.describe_plan(rows, cols)}), flush=True)
            except Exception as e:  # noqa: BLE001
                print(json.dumps({"shape": [rows, cols], "variant": tag, "error": str(e)}))
            for k in tun:
                _native.set_tuning(k, {"path": -1, "k1m": 1}.get(k, 0))


if __name__ == "__main__":
    main()
