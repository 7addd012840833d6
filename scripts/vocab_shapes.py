#!/usr/bin/env python
"""LLM-style shapes (batch x vocabulary): default plan, latency per call and
effective GB/s, against this library's copy kernel of the same bytes."""

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


def main():
    s = torch.cuda.Stream()
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    for rows, C in ((1, 32000), (8, 50257), (32, 151936), (64, 128256), (256, 32000),
                    (1024, 50257), (4096, 32000), (4096, 128256)):
        spec = configs.InputSpec(f"v{rows}x{C}", rows, C, "normal", 5, sigma=3.0)
        x0 = torch.from_numpy(configs.generate(spec)).cuda()
        R = max(2, -(-3 * l2 // (8 * rows * C)))
        xs = [x0] + [x0.clone() for _ in range(R - 1)]
        ys = [torch.empty_like(x0) for _ in range(R)]
        cu = copy_us(xs, ys, rows * C, 20, s)
        variants = [("default", {})] + ([("k3c", {"k3_impl": 5}), ("split", {"path": 2})]
                                        if len(sys.argv) > 1 else [])
        for tag, tun in variants:
            for k, v in tun.items():
                _native.set_tuning(k, v)
            try:
                us = bench_once(xs, ys, rows, C, 200, s)
                print(json.dumps({"rows": rows, "cols": C, "variant": tag,
                                  "plan": _native.describe_plan(rows, C)[:40],
                                  "us": round(us, 2), "gbs": round(8.0 * rows * C / us / 1e3),
                                  "copy_us": round(cu, 2), "vs_copy": round(cu / us, 3)}),
                      flush=True)
            except Exception as e:  # noqa: BLE001
                print(json.dumps({"rows": rows, "cols": C, "variant": tag, "error": str(e)[:80]}))
            _native.set_tuning("k3_impl", 3)
            _native.set_tuning("path", -1)


if __name__ == "__main__":
    main()
