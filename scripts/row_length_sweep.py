#!/usr/bin/env python
"""The default plan across row lengths at a fixed problem size (64 MiB in,
64 MiB out; rows = 16 Mi elements / C), against this library's own streaming
copy of the same bytes on the same buffers.  One JSON line per C."""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "scripts"))

import torch  # noqa: E402

from paper_1904_12380_b200 import _native, configs  # noqa: E402
from sweep import bench_once  # noqa: E402


def copy_us(xs, ys, n, reps, s):
    L = _native.lib()
    R = len(xs)

    def go(i):
        _native.check(L.sk_copy_f32(xs[i % R].data_ptr(), ys[i % R].data_ptr(), n, 0, s.cuda_stream))

    with torch.cuda.stream(s):
        for i in range(5):
            go(i)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(R * 8):
                go(i)
        g.replay()
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
    s.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * R * 8)


def main():
    total = 16 << 20
    s = torch.cuda.Stream()
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    cs = (50, 128, 256, 512, 1000, 1024, 1536, 2048, 3072, 4096, 6144, 8192, 12288, 16384,
          32768, 65536, 131072, 262144, 524288, 1048576, 2097152)
    if len(sys.argv) > 1:  # C,C,...
        cs = tuple(map(int, sys.argv[1].split(",")))
    for C in cs:
        rows = max(8, total // C)
        spec = configs.InputSpec(f"len{C}", rows, C, "normal", 7, sigma=4.0)
        x0 = torch.from_numpy(configs.generate(spec)).cuda()
        R = max(2, -(-3 * l2 // (8 * rows * C)))
        xs = [x0] + [x0.clone() for _ in range(R - 1)]
        ys = [torch.empty_like(x0) for _ in range(R)]
        us = bench_once(xs, ys, rows, C, 100, s)
        cu = copy_us(xs, ys, rows * C, 20, s)
        print(json.dumps({"cols": C, "rows": rows, "plan": _native.describe_plan(rows, C),
                          "us": us, "gbs": 8.0 * rows * C / us / 1e3,
                          "copy_us": cu, "vs_copy": cu / us}), flush=True)
        del xs, ys, x0


if __name__ == "__main__":
    main()
