#!/usr/bin/env python
"""End-to-end host-buffer path on reference-style pageable buffers: time per
call vs host copy threads and chunk size; plus the raw host memcpy rate and
the cost of page-locking the caller's buffers (cudaHostRegister), the two
alternatives to staging.  One JSON line per measurement.

    python scripts/e2e_pageable_probe.py --config c5a
"""

import argparse
import ctypes
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1904_12380_b200 as sk  # noqa: E402
from paper_1904_12380_b200 import _native, configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5a")
    ap.add_argument("--threads", default="1,2,4,8,12,16")
    ap.add_argument("--chunks", default="0,8192,65536")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--nt", default="1")
    args = ap.parse_args()
    spec = configs.get(args.config)
    x = configs.generate(spec)
    m = sk.alloc_matrix(*x.shape)
    m.view2d[:] = x
    o = sk.alloc_matrix(*x.shape)
    byts = 8.0 * x.size
    V = sk.KernelVariant.REFERENCE_CLIPPED
    sk.softmax(m, V, out=o)
    sets = [(c, t, n) for c in map(int, args.chunks.split(","))
            for t in map(int, args.threads.split(",")) for n in map(int, args.nt.split(","))]
    for ck, th, nt in sets:
        _native.set_tuning("host_nt", nt)
        _native.set_tuning("host_chunk_kb", ck)
        _native.set_tuning("host_threads", th)
        sk.softmax(m, V, out=o)
        t0 = time.perf_counter()
        for _ in range(args.reps):
            sk.softmax(m, V, out=o)
        dt = (time.perf_counter() - t0) / args.reps
        print(json.dumps({"what": "e2e pageable", "config": spec.name, "chunk_kb": ck,
                          "threads": th, "nt": nt, "ms": round(dt * 1e3, 2),
                          "gbs": round(byts / dt / 1e9, 1)}), flush=True)
    _native.set_tuning("host_chunk_kb", 0)
    _native.set_tuning("host_threads", 0)
    _native.set_tuning("host_nt", 1)
    # raw host copy rate (numpy, one thread) and page-locking cost
    dst = np.empty_like(x)
    t0 = time.perf_counter()
    np.copyto(dst, x)
    dt = time.perf_counter() - t0
    print(json.dumps({"what": "numpy copy 1 thread", "gbs": round(x.nbytes / dt / 1e9, 1)}))
    cudart = ctypes.CDLL("libcudart.so.12") if Path("/usr/local/cuda/lib64/libcudart.so.12").exists() \
        else None
    if cudart is not None:
        buf = np.empty_like(x)
        buf[:] = 0
        t0 = time.perf_counter()
        r1 = cudart.cudaHostRegister(ctypes.c_void_p(buf.ctypes.data), ctypes.c_size_t(buf.nbytes), 0)
        t1 = time.perf_counter()
        r2 = cudart.cudaHostUnregister(ctypes.c_void_p(buf.ctypes.data))
        t2 = time.perf_counter()
        print(json.dumps({"what": "cudaHostRegister", "bytes": buf.nbytes, "rc": [r1, r2],
                          "register_ms": round((t1 - t0) * 1e3, 1),
                          "unregister_ms": round((t2 - t1) * 1e3, 1)}))
    # pinned reference point
    mp = sk.Matrix2D.from_array(x, pinned=True)
    op = sk.alloc_matrix(*x.shape, pinned=True)
    sk.softmax(mp, V, out=op)
    t0 = time.perf_counter()
    for _ in range(args.reps):
        sk.softmax(mp, V, out=op)
    dt = (time.perf_counter() - t0) / args.reps
    print(json.dumps({"what": "e2e pinned", "ms": round(dt * 1e3, 2),
                      "gbs": round(byts / dt / 1e9, 1)}))


if __name__ == "__main__":
    torch.cuda.init()
    main()
