"""End to end through softmax(Matrix2D, out=) on the small configs (c1, c2,
c3): per-call time over repeated calls on the same buffers, pageable
(alloc_matrix) and page-locked up front.  Usage: python scripts/e2e_small_probe.py [out.jsonl]"""
import json
import statistics
import sys
import time

sys.path.insert(0, ".")
import paper_1904_12380_b200 as sk  # noqa: E402
from paper_1904_12380_b200 import configs, hostpin  # noqa: E402

out = open(sys.argv[1], "w") if len(sys.argv) > 1 else sys.stdout
V = sk.KernelVariant.REFERENCE_CLIPPED
for name in ("c1", "c2", "c3"):
    x = configs.generate(name)
    for kind in ("pageable", "pinned"):
        m = sk.Matrix2D.from_array(x, pinned=(kind == "pinned"))
        o = sk.alloc_matrix(*x.shape, pinned=(kind == "pinned"))
        for _ in range(5):
            sk.softmax(m, V, out=o)
        ts = []
        for _ in range(50):
            t0 = time.perf_counter()
            sk.softmax(m, V, out=o)
            ts.append((time.perf_counter() - t0) * 1e6)
        out.write(json.dumps({"config": name, "buffers": kind, "us_median": round(statistics.median(ts), 1),
                              "us_min": round(min(ts), 1), "gbs_median": round(8.0 * x.size / statistics.median(ts) / 1e3, 2),
                              "locked_by_library": hostpin.stats()["ranges"]}) + "\n")
        out.flush()
        del m, o
