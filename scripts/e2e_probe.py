#!/usr/bin/env python
"""PCIe ceilings and the host-buffer softmax (sk_softmax_f32_host) by chunk size."""

import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_1904_12380_b200 as sk  # noqa: E402
from paper_1904_12380_b200 import _native, configs  # noqa: E402


def gbs(nbytes, sec):
    return nbytes / sec / 1e9


def main():
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c2,c4")
    ap.add_argument("--chunks-kb", default="0,2048,4096,8192,16384,32768",
                    help="host_chunk_kb values (0 = auto)")
    ap.add_argument("--zero-copy", action="store_true", help="also time the zero-copy path")
    args = ap.parse_args()
    n = 64 << 20  # 64 MiB
    h = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
    h2 = torch.empty_like(h, pin_memory=True)
    d = torch.empty(n // 4, dtype=torch.float32, device="cuda")
    d2 = torch.empty_like(d)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        d.copy_(h, non_blocking=True)
        h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    res = {}
    t = time.perf_counter()
    for _ in range(10):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    res["h2d_GBps"] = gbs(10 * n, time.perf_counter() - t)
    t = time.perf_counter()
    for _ in range(10):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    res["d2h_GBps"] = gbs(10 * n, time.perf_counter() - t)
    t = time.perf_counter()
    for _ in range(10):
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    res["bidir_GBps_total"] = gbs(20 * n, time.perf_counter() - t)
    # two streams per direction, half the bytes each (more copy engines busy?)
    s3, s4 = torch.cuda.Stream(), torch.cuda.Stream()
    hh, hh2, dh, dh2 = h.view(2, -1), h2.view(2, -1), d.view(2, -1), d2.view(2, -1)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        for i, (sa, sb) in enumerate(((s1, s2), (s3, s4))):
            with torch.cuda.stream(sa):
                dh[i].copy_(hh[i], non_blocking=True)
            with torch.cuda.stream(sb):
                hh2[i].copy_(dh2[i], non_blocking=True)
    torch.cuda.synchronize()
    res["bidir_2x2_GBps_total"] = gbs(20 * n, time.perf_counter() - t)
    t = time.perf_counter()
    for _ in range(10):
        for i, sa in enumerate((s1, s3)):
            with torch.cuda.stream(sa):
                dh[i].copy_(hh[i], non_blocking=True)
    torch.cuda.synchronize()
    res["h2d_2streams_GBps"] = gbs(10 * n, time.perf_counter() - t)
    print(json.dumps(res), flush=True)
    for name in args.configs.split(","):
        spec = configs.get(name)
        m = sk.Matrix2D.from_array(configs.generate(spec), pinned=True)
        out = sk.alloc_matrix(spec.rows, spec.cols, pinned=True)
        cases = [(0, int(k)) for k in args.chunks_kb.split(",")]
        if args.zero_copy:
            cases.insert(0, (1, 0))
        for zc, kb in cases:
            _native.set_tuning("host_zero_copy", zc)
            _native.set_tuning("host_chunk_kb", kb)
            sk.softmax(m, sk.KernelVariant.REFERENCE_CLIPPED, out=out)
            reps = 10
            t = time.perf_counter()
            for _ in range(reps):
                sk.softmax(m, sk.KernelVariant.REFERENCE_CLIPPED, out=out)
            dt = (time.perf_counter() - t) / reps
            ok = bool((out.view2d == sk.softmax(torch.from_numpy(m.view2d).cuda(),
                       sk.KernelVariant.REFERENCE_CLIPPED).cpu().numpy()).all())
            print(json.dumps({"config": name, "zero_copy": zc, "chunk_kb": kb, "ms": dt * 1e3,
                              "bitwise_equal_device": ok,
                              "e2e_GBps": gbs(8 * spec.rows * spec.cols, dt)}), flush=True)
    _native.set_tuning("host_chunk_kb", 0)
    _native.set_tuning("host_zero_copy", 0)


if __name__ == "__main__":
    main()
