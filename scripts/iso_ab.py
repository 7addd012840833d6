#!/usr/bin/env python
"""Single-launch (isolated) and back-to-back (steady) device time of the
softmax for tuning-knob sets, on BASELINE-config or arbitrary shapes.

    python scripts/iso_ab.py --shapes c2,c3,16384x1000 --sets "default;k1b=0;k1b_w=16"

isolated: each launch is bracketed by its own event pair on a stream parked
behind a device sleep (so host launch latency is not timed), with a device
sleep between launches (no PDL overlap with a predecessor); inputs rotate
over buffer pairs spanning >= 3x L2, so every launch reads cold HBM and the
previous launches' outputs are still dirty in L2, as for a drop-in call.
steady: a CUDA graph of back-to-back launches over the same rotation.
Each set's output is compared bitwise with the first set's.  One JSON line
per (shape, set).
"""

import argparse
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "scripts"))

import torch  # noqa: E402

from paper_1904_12380_b200 import _native, configs  # noqa: E402

DEFAULTS = {"k1_threads": 128, "grid_mult": 0, "path": -1, "k1_pf": -1, "pdl": 1, "k1_lpr": 0,
            "k1_nv": 0, "k1_u": 0}


def parse_sets(s):
    out = []
    for part in s.split(";"):
        part = part.strip()
        if not part or part == "default":
            out.append(("default", {}))
            continue
        kv = dict((k, int(v)) for k, v in (t.split("=") for t in part.split(",")))
        bad = set(kv) - set(DEFAULTS)
        if bad:
            raise SystemExit(f"no default recorded for {sorted(bad)}")
        out.append((part, kv))
    return out


def shape_input(tok):
    if tok.startswith("c"):
        spec = configs.get(tok)
        return tok, configs.generate(spec)
    rows, cols = map(int, tok.split("x"))
    spec = configs.InputSpec(f"k{rows}x{cols}", rows, cols, "normal", 11, sigma=4.0)
    return tok, configs.generate(spec)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="c2,c3")
    ap.add_argument("--sets", default="default;k1b=0")
    ap.add_argument("--iso", type=int, default=60)
    ap.add_argument("--steady", type=int, default=600)
    args = ap.parse_args()
    L = _native.lib()
    s = torch.cuda.Stream()
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    flag = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    for tok in args.shapes.split(","):
        name, xh = shape_input(tok)
        rows, cols = xh.shape
        x0 = torch.from_numpy(xh).cuda()
        R = max(2, -(-3 * l2 // (8 * rows * cols)))
        xs = [x0] + [x0.clone() for _ in range(R - 1)]
        ys = [torch.empty_like(x0) for _ in range(R)]
        base = None
        for tag, kv in parse_sets(args.sets):
            for k, v in DEFAULTS.items():
                _native.set_tuning(k, kv.get(k, v))

            def launch(i):
                _native.check(L.sk_softmax_f32(xs[i % R].data_ptr(), ys[i % R].data_ptr(), rows,
                                               cols, cols, cols, 0, flag.data_ptr(), None, 0,
                                               s.cuda_stream))

            rec = {"shape": name, "rows": rows, "cols": cols, "set": tag}
            try:
                rec["plan"] = _native.describe_plan(rows, cols)
                with torch.cuda.stream(s):
                    for i in range(2 * R):
                        launch(i)
                s.synchronize()
                out = ys[(2 * R - 1) % R].clone()
                if base is None:
                    base = out
                rec["bits_equal_first"] = bool(torch.equal(out.view(torch.int32),
                                                           base.view(torch.int32)))
                # isolated
                n = args.iso
                ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                      for _ in range(n)]
                with torch.cuda.stream(s):
                    torch.cuda._sleep(int(2e5 + n * 1.5e5))
                    for i in range(n):
                        torch.cuda._sleep(20000)  # ~10 us gap: no overlap with a predecessor
                        ev[i][0].record(s)
                        launch(i)
                        ev[i][1].record(s)
                s.synchronize()
                iso = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
                # steady (graph of back-to-back launches)
                G = R * max(1, 64 // R)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.stream(s):
                    with torch.cuda.graph(g, stream=s):
                        for i in range(G):
                            launch(i)
                    g.replay()
                s.synchronize()
                reps = max(1, args.steady // G)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(s):
                    e0.record(s)
                    for _ in range(reps):
                        g.replay()
                    e1.record(s)
                s.synchronize()
                steady = e0.elapsed_time(e1) * 1e3 / (reps * G)
                byts = 8.0 * rows * cols
                rec.update(iso_med_us=round(statistics.median(iso), 3), iso_min_us=round(iso[0], 3),
                           iso_mean_us=round(statistics.fmean(iso), 3),
                           iso_gbs=round(byts / statistics.median(iso) / 1e3, 1),
                           steady_us=round(steady, 3), steady_gbs=round(byts / steady / 1e3, 1))
            except Exception as e:  # noqa: BLE001
                rec["error"] = str(e)
            print(json.dumps(rec), flush=True)
        for k, v in DEFAULTS.items():
            _native.set_tuning(k, v)
        # copy of the same bytes, isolated, for scale
        n = rows * cols
        if n % 4 == 0:
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(args.iso)]
            with torch.cuda.stream(s):
                torch.cuda._sleep(int(2e5 + args.iso * 1.5e5))
                for i in range(args.iso):
                    torch.cuda._sleep(20000)
                    ev[i][0].record(s)
                    _native.check(L.sk_copy_f32(xs[i % R].data_ptr(), ys[i % R].data_ptr(), n, 0,
                                                s.cuda_stream))
                    ev[i][1].record(s)
            s.synchronize()
            iso = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
            print(json.dumps({"shape": name, "set": "own copy kernel", "iso_med_us":
                              round(statistics.median(iso), 3)}), flush=True)
        del xs, ys, x0
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
