#!/usr/bin/env python
"""Where the host-buffer path's time goes on c2 (33.5 MB each way): PCIe
transfers of the same bytes under different dependency structures, against
softmax(Matrix2D).  One JSON line per variant (median of reps, wall clock
around a synchronised region)."""

import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_1904_12380_b200 as sk  # noqa: E402
from paper_1904_12380_b200 import configs  # noqa: E402


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    return statistics.median(ts) * 1e6


def main():
    spec = configs.get(sys.argv[1] if len(sys.argv) > 1 else "c2")
    n = spec.rows * spec.cols
    hx = torch.empty(n, dtype=torch.float32, pin_memory=True)
    hy = torch.empty(n, dtype=torch.float32, pin_memory=True)
    dx = torch.empty(n, dtype=torch.float32, device="cuda")
    dy = torch.empty(n, dtype=torch.float32, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}

    def both_whole():
        with torch.cuda.stream(s1):
            dx.copy_(hx, non_blocking=True)
        with torch.cuda.stream(s2):
            hy.copy_(dy, non_blocking=True)

    def chunks(k):
        b = (n + k - 1) // k
        return [(i * b, min(n, (i + 1) * b)) for i in range(k)]

    def both_chunked(k):
        def f():
            for a, e in chunks(k):
                with torch.cuda.stream(s1):
                    dx[a:e].copy_(hx[a:e], non_blocking=True)
                with torch.cuda.stream(s2):
                    hy[a:e].copy_(dy[a:e], non_blocking=True)
        return f

    def pipelined(k):
        evs = [torch.cuda.Event() for _ in range(k)]

        def f():
            for i, (a, e) in enumerate(chunks(k)):
                with torch.cuda.stream(s1):
                    dx[a:e].copy_(hx[a:e], non_blocking=True)
                    evs[i].record(s1)
                with torch.cuda.stream(s2):
                    s2.wait_event(evs[i])
                    hy[a:e].copy_(dx[a:e], non_blocking=True)
        return f

    out["h2d_only_us"] = timeit(lambda: dx.copy_(hx, non_blocking=True))
    out["d2h_only_us"] = timeit(lambda: hy.copy_(dy, non_blocking=True))
    out["both_whole_us"] = timeit(both_whole)
    for k in (4, 8, 16):
        out[f"both_chunked{k}_us"] = timeit(both_chunked(k))
        out[f"pipelined{k}_us"] = timeit(pipelined(k))
    m_in = sk.Matrix2D.from_array(configs.generate(spec), pinned=True)
    m_out = sk.alloc_matrix(spec.rows, spec.cols, pinned=True)
    out["softmax_host_us"] = timeit(lambda: sk.softmax(m_in, sk.KernelVariant.REFERENCE_CLIPPED, out=m_out))
    out["bytes_each_way"] = 4 * n
    print(json.dumps({k: (round(v, 1) if isinstance(v, float) else v) for k, v in out.items()}), flush=True)


if __name__ == "__main__":
    main()
