"""cudaHostRegister time vs the range's size / alignment (why the reference's
np.zeros(n + pad) buffers register 4x slower than an exact 2 GiB array).
Usage: python scripts/hostreg_align_probe.py [out.jsonl]"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1904_12380_b200 import _native  # noqa: E402

L = _native.lib()
out = open(sys.argv[1], "w") if len(sys.argv) > 1 else sys.stdout
import torch  # noqa: E402

torch.zeros(1, device="cuda")


def reg(tag, ptr, n, **kw):
    best = None
    for _ in range(2):
        t0 = time.perf_counter()
        st = L.sk_host_register(ptr, n)
        t1 = time.perf_counter()
        if st == 0:
            L.sk_host_unregister(ptr)
        ms = (t1 - t0) * 1e3
        best = ms if best is None else min(best, ms)
    out.write(json.dumps({"case": tag, "ptr_mod_2m": ptr % (2 << 20), "ptr_mod_4k": ptr % 4096,
                          "bytes": n, "bytes_mod_2m": n % (2 << 20), "status": st,
                          "register_ms": round(best, 2), **kw}) + "\n")
    out.flush()


G2 = 1 << 31
M2 = 2 << 20
a = np.zeros(G2 // 4, np.float32)
a[:] = 1
b = np.zeros(G2 // 4 + 8, np.float32)
b[:] = 1
pa, pb = a.ctypes.data, b.ctypes.data
reg("exact 2 GiB array, as is", pa, a.nbytes)
reg("2 GiB + 32 B array, as is", pb, b.nbytes)
reg("2 GiB + 32 B array, first 2 GiB", pb, G2)
reg("2 GiB + 32 B array, +32 B .. 2 GiB", pb + 32, G2)
reg("2 GiB + 32 B array, minus the last 4 KiB", pb, b.nbytes - 4096)
reg("exact array, 2 GiB - 4 KiB", pa, G2 - 4096)
reg("exact array, 2 GiB - 2 MiB", pa, G2 - M2)
ia = (pb + M2 - 1) // M2 * M2
ib = (pb + b.nbytes) // M2 * M2
reg("2 GiB + 32 B array, inner 2 MiB-aligned window", ia, ib - ia)
ia4 = (pb + 4095) // 4096 * 4096
ib4 = (pb + b.nbytes) // 4096 * 4096
reg("2 GiB + 32 B array, inner 4 KiB-aligned window", ia4, ib4 - ia4)
reg("1 GiB of the exact array", pa, G2 // 2)
reg("1 GiB + 4 KiB of the exact array", pa, G2 // 2 + 4096)
reg("1.5 GiB of the exact array", pa, G2 // 4 * 3)
c = np.zeros((3 << 30) // 4, np.float32)
c[:] = 1
reg("exact 3 GiB array", c.ctypes.data, c.nbytes)
reg("exact 3 GiB array, first 2 GiB", c.ctypes.data, G2)
reg("exact 3 GiB array, first 2 GiB + 32 B", c.ctypes.data, G2 + 32)
reg("exact 3 GiB array, first 2 GiB + 2 MiB", c.ctypes.data, G2 + M2)
