"""Host path (sk_softmax_f32_host) on c5a by how the caller's buffers are
page-locked: cudaHostAlloc, registered in place at a 2 MiB-aligned address,
registered at the reference's alloc_matrix alignment (32 B).
Usage: python scripts/hostreg_dma_probe.py [out.jsonl]"""
import ctypes
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1904_12380_b200 as sk  # noqa: E402
from paper_1904_12380_b200 import _native, configs, hostpin  # noqa: E402

L = _native.lib()
out = open(sys.argv[1], "w") if len(sys.argv) > 1 else sys.stdout
hostpin.configure(enabled=False)
x = configs.generate("c5a")
rows, cols = x.shape
M2 = 2 << 20


def run(tag, xin, yout, **kw):
    bad = ctypes.c_int64(-1)
    ts = []
    for _ in range(6):
        t0 = time.perf_counter()
        st = L.sk_softmax_f32_host(xin.ctypes.data, yout.ctypes.data, rows, cols, 0, 0,
                                   ctypes.byref(bad))
        ts.append((time.perf_counter() - t0) * 1e3)
        assert st == 0
    out.write(json.dumps({"case": tag, "ms": [round(t, 2) for t in ts],
                          "gbs_best": round(8.0 * x.size / min(ts[1:]) / 1e6, 1), **kw}) + "\n")
    out.flush()


def carve(off):
    raw = np.zeros(x.size + (2 * M2 + 64) // 4, np.float32)
    start = (-raw.ctypes.data) % M2 + off
    v = raw[start // 4: start // 4 + x.size]
    return raw, v


pi = sk.Matrix2D.from_array(x, pinned=True)
po = sk.alloc_matrix(rows, cols, pinned=True)
run("cudaHostAlloc in / out", pi.data, po.data)
for off in (0, 32, 4096):
    ra, a = carve(off)
    rb, b = carve(off)
    a[:] = x.ravel()
    b[:] = 0
    lo = lambda r: (r.ctypes.data + M2 - 1) // M2 * M2  # noqa: E731
    hi = lambda r: (r.ctypes.data + r.nbytes) // M2 * M2  # noqa: E731
    t0 = time.perf_counter()
    assert L.sk_host_register(lo(ra), hi(ra) - lo(ra)) == 0
    assert L.sk_host_register(lo(rb), hi(rb) - lo(rb)) == 0
    treg = (time.perf_counter() - t0) * 1e3
    run(f"registered in place, data at 2 MiB + {off} B", a, b, register_ms=round(treg, 1))
    run("registered input, cudaHostAlloc output", a, po.data)
    run("cudaHostAlloc input, registered output", pi.data, b)
    L.sk_host_unregister(lo(ra))
    L.sk_host_unregister(lo(rb))
    del ra, rb, a, b
