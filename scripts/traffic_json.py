#!/usr/bin/env python
"""Build traffic.json (what bench.py reports as roofline.traffic) from the ncu
CSVs written by scripts/traffic_run.sh: per config, the median per-launch
dram__bytes_read/write of the default plan's kernel(s), with that plan's
description (computed here, on the GPU box) so bench.py only uses a number
measured for the plan it runs.  Usage: traffic_json.py <csv dir> <out json>."""

import csv
import json
import statistics
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1904_12380_b200 import _native, configs  # noqa: E402


def parse(path):
    rows = defaultdict(dict)
    with open(path, newline="") as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        key = r["ID"]
        rows[key]["kernel"] = r["Kernel Name"]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        if r["Metric Name"].startswith("dram__bytes"):
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        elif r["Metric Name"] == "gpu__time_duration.sum":
            v *= {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
        rows[key][r["Metric Name"]] = v
    return list(rows.values())


def main():
    src, out = Path(sys.argv[1]), Path(sys.argv[2])
    res = {"_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch of the default "
                    "plan's kernel(s), ncu --cache-control none --clock-control none, launches "
                    "11-20 of bench.py's loop (steady state, rotating buffers). Algorithmic = "
                    "8 B/element. Built by scripts/traffic_json.py from the ncu CSVs of scripts/r2_profiles.sh (profiles/r2_traffic_<config>.csv)"}
    for c in ("c1", "c2", "c3", "c5a", "c4", "c5b"):
        p = src / f"traffic_{c}.csv"
        if not p.exists():
            continue
        launches = parse(p)
        if not launches:
            continue
        spec = configs.get(c)
        rd = statistics.median(l.get("dram__bytes_read.sum", 0.0) for l in launches)
        wr = statistics.median(l.get("dram__bytes_write.sum", 0.0) for l in launches)
        res[c] = {
            "plan": _native.describe_plan(spec.rows, spec.cols),
            "kernel": launches[0]["kernel"][:64],
            "dram_read_bytes": rd,
            "dram_write_bytes": wr,
            "dram_bytes_per_launch": rd + wr,
            "algorithmic_bytes": 8.0 * spec.rows * spec.cols,
            "ncu_duration_ns_median": statistics.median(
                l.get("gpu__time_duration.sum", 0.0) for l in launches),
        }
    out.write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps({k: v.get("dram_bytes_per_launch") if isinstance(v, dict) else None
                      for k, v in res.items()}))


if __name__ == "__main__":
    main()
