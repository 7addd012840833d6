#!/usr/bin/env python
"""Host cost of one drop-in call on a small job (c1 = [4096, 50]): wall time
per call, back to back, of the raw C entry point through ctypes, of
softmax_into (async) and of softmax (allocates, checks the non-finite flag --
a stream sync).  One JSON line per path.

    python scripts/call_overhead.py [--config c1] [--calls 3000]
"""

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_1904_12380_b200 as sk  # noqa: E402
from paper_1904_12380_b200 import _native, configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--calls", type=int, default=3000)
    args = ap.parse_args()
    x = torch.from_numpy(configs.generate(args.config)).cuda()
    y = torch.empty_like(x)
    rows, cols = x.shape
    L = _native.lib()
    flag = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    V = sk.KernelVariant.REFERENCE_CLIPPED

    def raw():
        L.sk_softmax_f32(x.data_ptr(), y.data_ptr(), rows, cols, cols, cols, 0, flag.data_ptr(),
                         None, 0, s)

    paths = {"C ABI via ctypes": raw,
             "softmax_into(check_finite=False)": lambda: sk.softmax_into(x, y, V,
                                                                          check_finite=False),
             "softmax (checked: syncs)": lambda: sk.softmax(x, V)}
    for name, fn in paths.items():
        for _ in range(50):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.calls):
            fn()
        torch.cuda.synchronize()
        us = (time.perf_counter() - t0) / args.calls * 1e6
        print(json.dumps({"config": args.config, "path": name, "us_per_call": round(us, 2)}),
              flush=True)


if __name__ == "__main__":
    main()
