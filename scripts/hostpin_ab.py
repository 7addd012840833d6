"""softmax(pageable Matrix2D, out=pageable) on c5a, repeated calls, by page-
locking policy: edges registered or staged, device slots at the host page
phase or not.  Usage: python scripts/hostpin_ab.py [out.jsonl]"""
import gc
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1904_12380_b200 as sk  # noqa: E402
from paper_1904_12380_b200 import _native, configs, hostpin  # noqa: E402

out = open(sys.argv[1], "w") if len(sys.argv) > 1 else sys.stdout
name = sys.argv[2] if len(sys.argv) > 2 else "c5a"
x = configs.generate(name)
import torch  # noqa: E402

ref = sk.softmax(torch.from_numpy(x).cuda(), sk.KernelVariant.REFERENCE_CLIPPED).cpu().numpy()
for edges in (False, True):
    for phase in (0,):  # host_phase 1 (device slot at the host page phase) was removed: no gain
        hostpin.configure(enabled=True, edges=edges, min_bytes=16 << 20)
        m = sk.alloc_matrix(*x.shape)
        m.view2d[:] = x
        o = sk.alloc_matrix(*x.shape)
        ts = []
        for i in range(8):
            t0 = time.perf_counter()
            sk.softmax(m, sk.KernelVariant.REFERENCE_CLIPPED, out=o)
            ts.append((time.perf_counter() - t0) * 1e3)
        ok = bool(np.array_equal(o.view2d.view(np.uint32), ref.view(np.uint32)))
        out.write(json.dumps({"config": name, "edges": edges, "host_phase": phase,
                              "ms": [round(t, 2) for t in ts],
                              "gbs_steady": round(8.0 * x.size / min(ts[2:]) / 1e6, 1),
                              "bitwise_equal_device_path": ok, "stats": hostpin.stats()}) + "\n")
        out.flush()
        del m, o
        gc.collect()
