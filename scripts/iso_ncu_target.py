#!/usr/bin/env python
"""ncu target: single launches (synchronised one by one) of the softmax and of
copy kernels at several sizes, for gpu__time_duration of an isolated launch.

    ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none \\
        --csv --log-file out.csv python scripts/iso_ncu_target.py --manifest m.json

Each item launches `--reps` times on rotating buffers (>= 3x L2 of bytes, so
inputs are cold in L2 and earlier outputs are still dirty there, as for a
drop-in call), with a device synchronise after every launch.  The manifest
lists items in launch order with their launch counts, so the ncu CSV rows can
be attributed (scripts/iso_ncu_parse.py).
"""

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_1904_12380_b200 import _native, configs  # noqa: E402

KNOB_DEFAULTS = {"grid_mult": 0, "k1_threads": 128, "k1_pf": -1, "k1_lpr": 0, "k1_nv": 0,
                 "k1_u": 0}


def items_default():
    out = []
    for mb in (1, 4, 16, 64, 256, 1024):
        out.append({"kind": "copy", "bytes": mb << 20})
        out.append({"kind": "torch_copy", "bytes": mb << 20})
    out.append({"kind": "empty"})
    for shp in ("4096x128", "16384x128", "65536x128", "262144x128", "1048576x128"):
        out.append({"kind": "softmax", "shape": shp, "knobs": {}})
    for shp in ("c1", "c2", "c3"):
        out.append({"kind": "softmax", "shape": shp, "knobs": {}})
    u2 = {"k1_lpr": 8, "k1_nv": 4, "k1_u": 2}
    for kn in ({"grid_mult": 1}, {"grid_mult": 2}, {"grid_mult": 1, "k1_pf": 1},
               {"grid_mult": 2, "k1_pf": 1}, {"k1_threads": 256}, {"k1_threads": 64}, u2,
               {**u2, "grid_mult": 1}, {**u2, "grid_mult": 2}):
        out.append({"kind": "softmax", "shape": "c2", "knobs": kn})
    for kn in ({"grid_mult": 1}, {"grid_mult": 2}, {"grid_mult": 1, "k1_pf": 1},
               {"grid_mult": 2, "k1_pf": 1}, {"k1_threads": 256}, {"k1_threads": 64}):
        out.append({"kind": "softmax", "shape": "c3", "knobs": kn})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--manifest", required=True)
    ap.add_argument("--reps", type=int, default=8)
    ap.add_argument("--items", default="")
    args = ap.parse_args()
    items = json.loads(args.items) if args.items else items_default()
    L = _native.lib()
    dev = torch.device("cuda", 0)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flag = torch.full((1,), -1, dtype=torch.int64, device=dev)
    s = torch.cuda.current_stream()
    manifest = []
    for it in items:
        if it["kind"] == "empty":
            for _ in range(args.reps):
                torch.cuda._sleep(1)
                torch.cuda.synchronize()
            manifest.append({**it, "launches": args.reps, "kernels_per_launch": 1})
            continue
        if it["kind"] in ("copy", "torch_copy"):
            n = it["bytes"] // 8  # bytes = read + write
            R = max(2, -(-3 * l2 // (8 * n)))
            xs = [torch.zeros(n, dtype=torch.float32, device=dev) for _ in range(R)]
            ys = [torch.empty_like(xs[0]) for _ in range(R)]
            for i in range(args.reps + R):
                if it["kind"] == "copy":
                    _native.check(L.sk_copy_f32(xs[i % R].data_ptr(), ys[i % R].data_ptr(), n, 0,
                                                s.cuda_stream))
                else:
                    ys[i % R].copy_(xs[i % R])
                torch.cuda.synchronize()
            manifest.append({**it, "launches": args.reps + R, "skip": R, "kernels_per_launch": 1})
            del xs, ys
            continue
        tok = it["shape"]
        if tok.startswith("c"):
            xh = configs.generate(configs.get(tok))
        else:
            r, c = map(int, tok.split("x"))
            xh = configs.generate(configs.InputSpec(f"k{tok}", r, c, "normal", 11, sigma=4.0))
        rows, cols = xh.shape
        for k, v in KNOB_DEFAULTS.items():
            try:
                _native.set_tuning(k, it["knobs"].get(k, v))
            except Exception:  # noqa: BLE001 -- knob absent in this build
                pass
        x0 = torch.from_numpy(xh).to(dev)
        R = max(2, -(-3 * l2 // (8 * rows * cols)))
        xs = [x0] + [x0.clone() for _ in range(R - 1)]
        ys = [torch.empty_like(x0) for _ in range(R)]
        plan = _native.describe_plan(rows, cols)
        for i in range(args.reps + R):
            _native.check(L.sk_softmax_f32(xs[i % R].data_ptr(), ys[i % R].data_ptr(), rows, cols,
                                           cols, cols, 0, flag.data_ptr(), None, 0, s.cuda_stream))
            torch.cuda.synchronize()
        manifest.append({**it, "plan": plan, "rows": rows, "cols": cols, "launches": args.reps + R,
                         "skip": R, "kernels_per_launch": 1})
        del xs, ys, x0
        torch.cuda.empty_cache()
    for k, v in KNOB_DEFAULTS.items():
        try:
            _native.set_tuning(k, v)
        except Exception:  # noqa: BLE001
            pass
    Path(args.manifest).write_text(json.dumps(manifest, indent=1))


if __name__ == "__main__":
    main()
