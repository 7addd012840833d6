"""Cost of page-locking a caller's pageable buffers in place (hostpin.py):
cudaHostRegister / Unregister of a touched np.zeros range by size, in one
call and split over host threads, and the host path before / after.
Usage: python scripts/hostpin_probe.py [out.jsonl]"""
import json
import sys
import threading
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1904_12380_b200 as sk  # noqa: E402
from paper_1904_12380_b200 import _native, hostpin  # noqa: E402

L = _native.lib()
out = open(sys.argv[1], "w") if len(sys.argv) > 1 else sys.stdout


def emit(**kw):
    out.write(json.dumps(kw) + "\n")
    out.flush()


import torch  # noqa: E402

torch.cuda.init()
torch.zeros(1, device="cuda")

for mib in (64, 256, 1024, 2048):
    a = np.zeros(mib << 18, np.float32)
    a[:] = 1.0
    for rep in range(2):
        t0 = time.perf_counter()
        st = L.sk_host_register(a.ctypes.data, a.nbytes)
        t1 = time.perf_counter()
        L.sk_host_unregister(a.ctypes.data)
        t2 = time.perf_counter()
        emit(what="register", mib=mib, rep=rep, status=st, register_ms=(t1 - t0) * 1e3,
             unregister_ms=(t2 - t1) * 1e3)
    for nthr in (4, 8, 16):
        part = (a.nbytes // nthr + 4095) // 4096 * 4096
        base = a.ctypes.data
        rngs = [(base + i * part, min(part, a.nbytes - i * part)) for i in range(nthr)
                if i * part < a.nbytes]
        res = [0] * len(rngs)

        def work(i):
            res[i] = L.sk_host_register(rngs[i][0], rngs[i][1])

        t0 = time.perf_counter()
        th = [threading.Thread(target=work, args=(i,)) for i in range(len(rngs))]
        [t.start() for t in th]
        [t.join() for t in th]
        t1 = time.perf_counter()
        for p, _ in rngs:
            L.sk_host_unregister(p)
        t2 = time.perf_counter()
        emit(what="register_split", mib=mib, threads=nthr, status=res, register_ms=(t1 - t0) * 1e3,
             unregister_ms=(t2 - t1) * 1e3)
    del a

from paper_1904_12380_b200 import configs  # noqa: E402

for name, rows in (("c5a", None), ("c2", None)):
    spec = configs.get(name)
    x = configs.generate(spec)
    m = sk.alloc_matrix(*x.shape)
    m.view2d[:] = x
    o = sk.alloc_matrix(*x.shape)
    byts = 8.0 * x.size
    ts = []
    for i in range(8):
        t0 = time.perf_counter()
        sk.softmax(m, sk.KernelVariant.REFERENCE_CLIPPED, out=o)
        ts.append((time.perf_counter() - t0) * 1e3)
    emit(what="calls", config=name, ms=[round(t, 2) for t in ts],
         gbs=[round(byts / t / 1e6, 1) for t in ts], stats=hostpin.stats())
    del m, o


def huge_kb(addr, nbytes):
    """AnonHugePages (kB) of the mappings overlapping [addr, addr + nbytes)."""
    tot, inside = 0, False
    for line in open("/proc/self/smaps"):
        f = line.split()
        if "-" in f[0] and len(f) >= 5 and not f[0].endswith(":"):
            lo, hi = (int(v, 16) for v in f[0].split("-"))
            inside = lo < addr + nbytes and hi > addr
        elif inside and f[0] == "AnonHugePages:":
            tot += int(f[1])
    return tot


# where the registration time goes in the call flow: the input (filled by one
# numpy copy) and the output (first touched by the staging threads)
hostpin.configure(enabled=False)
x = configs.generate("c5a")
m = sk.alloc_matrix(*x.shape)
m.view2d[:] = x
o = sk.alloc_matrix(*x.shape)
emit(what="huge_before_call", m_kb=huge_kb(m.data.ctypes.data, m.data.nbytes),
     o_kb=huge_kb(o.data.ctypes.data, o.data.nbytes))
sk.softmax(m, sk.KernelVariant.REFERENCE_CLIPPED, out=o)
emit(what="huge_after_call", m_kb=huge_kb(m.data.ctypes.data, m.data.nbytes),
     o_kb=huge_kb(o.data.ctypes.data, o.data.nbytes))
for name, a in (("m", m.data.base), ("o", o.data.base), ("x", x)):
    for rep in range(2):
        t0 = time.perf_counter()
        st = L.sk_host_register(a.ctypes.data, a.nbytes)
        t1 = time.perf_counter()
        L.sk_host_unregister(a.ctypes.data)
        t2 = time.perf_counter()
        emit(what="register_in_flow", buf=name, rep=rep, status=st, register_ms=(t1 - t0) * 1e3,
             unregister_ms=(t2 - t1) * 1e3, huge_kb=huge_kb(a.ctypes.data, a.nbytes))
