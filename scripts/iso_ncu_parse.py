#!/usr/bin/env python
"""Attribute an ncu launch list (gpu__time_duration.sum CSV) of
scripts/iso_ncu_target.py to its manifest items; one JSON line per item with
the median / min isolated duration and GB/s (8 B/element for softmax, the
item's read+write bytes for copies), plus a least-squares fit
t = a + bytes / BW over the copy items of each kind.

    python scripts/iso_ncu_parse.py launches.csv manifest.json
"""

import csv
import json
import re
import statistics
import sys

PAT = {
    "copy": re.compile(r"k_copy4"),
    "torch_copy": re.compile(r"copy_kernel|direct_copy|CopyFunctor|elementwise_kernel.*copy", re.I),
    "empty": re.compile(r"spin|sleep", re.I),
    "softmax": re.compile(r"k1_rows|k1b_rows|k1m_rows|k3_|k4_|k_seg"),
}


def rows_of(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    out = []
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            out.append((r["Kernel Name"], float(r["Metric Value"])))
    return out


def main():
    rows = rows_of(sys.argv[1])
    man = json.load(open(sys.argv[2]))
    i = 0
    fits = {}
    for it in man:
        if it["kind"] == "torch_copy":  # same-device copy_ is a cudaMemcpy: no kernel in ncu
            continue
        pat = PAT[it["kind"]]
        got = []
        while i < len(rows) and len(got) < it["launches"]:
            if pat.search(rows[i][0]):
                got.append(rows[i])
            i += 1
        d = [v for _, v in got[it.get("skip", 0):]]
        rec = {k: it[k] for k in it if k not in ("launches", "kernels_per_launch", "skip")}
        if d:
            med = statistics.median(d)
            rec.update(n=len(d), med_ns=med, min_ns=min(d), kernel=got[-1][0][:60])
            if it["kind"] in ("copy", "torch_copy"):
                rec["gbs"] = round(it["bytes"] / med, 1)
                fits.setdefault(it["kind"], []).append((it["bytes"], med))
            elif it["kind"] == "softmax":
                rec["gbs"] = round(8.0 * it["rows"] * it["cols"] / med, 1)
        print(json.dumps(rec))
    for kind, pts in fits.items():
        if len(pts) < 2:
            continue
        n = len(pts)
        mx = sum(b for b, _ in pts) / n
        my = sum(t for _, t in pts) / n
        sxx = sum((b - mx) ** 2 for b, _ in pts)
        sxy = sum((b - mx) * (t - my) for b, t in pts)
        slope = sxy / sxx
        print(json.dumps({"fit": kind, "intercept_ns": round(my - slope * mx, 1),
                          "marginal_gbs": round(1.0 / slope, 1), "points": pts}))


if __name__ == "__main__":
    main()
