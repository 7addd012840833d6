import json, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/scripts')
import torch
from paper_1904_12380_b200 import _native, configs
from sweep import bench_once
for rows, C in ((512, 262144), (1024, 1048576), (1024, 16384), (256, 32000), (64, 262144), (2048, 50257)):
    spec = configs.InputSpec(f"s{rows}x{C}", rows, C, "normal", 3, sigma=4.0)
    x0 = torch.from_numpy(configs.generate(spec)).cuda()
    R = max(2, -(-3 * (126 << 20) // (8 * rows * C)))
    xs = [x0] + [x0.clone() for _ in range(R - 1)]; ys = [torch.empty_like(x0) for _ in range(R)]
    s = torch.cuda.Stream()
    for cp in (0, 1, 0, 1):
        _native.set_tuning("coop_pdl", cp)
        us = bench_once(xs, ys, rows, C, 40 if rows * C > 1e8 else 200, s)
        print(json.dumps({"shape": [rows, C], "coop_pdl": cp, "us": round(us, 2), "plan": _native.describe_plan(rows, C)[:30]}), flush=True)
    _native.set_tuning("coop_pdl", 0)
