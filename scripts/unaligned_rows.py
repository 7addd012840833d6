import json, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/scripts')
import torch
from paper_1904_12380_b200 import _native, configs
from sweep import bench_once
for rows, C in ((16384, 1501), (8192, 3001), (4096, 5001), (4096, 8191), (2048, 50257),
                (512, 262147)):
    spec = configs.InputSpec(f"u{C}", rows, C, "normal", 3, sigma=4.0)
    x0 = torch.from_numpy(configs.generate(spec)).cuda()
    R = max(2, -(-3 * (126 << 20) // (8 * rows * C)))
    xs = [x0] + [x0.clone() for _ in range(R - 1)]; ys = [torch.empty_like(x0) for _ in range(R)]
    s = torch.cuda.Stream()
    for k1m in (1, 0):  # K1m 32-bit vs the split path it replaces
        _native.set_tuning("k1m", k1m)
        us = bench_once(xs, ys, rows, C, 50, s)
        print(json.dumps({"shape": [rows, C], "k1m": k1m, "plan": _native.describe_plan(rows, C),
                          "us": us, "gbs": 8.0 * rows * C / us / 1e3}))
    _native.set_tuning("k1m", 1)
