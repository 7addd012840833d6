#!/usr/bin/env python
"""Kernel-shape sweep on one GPU: device time per launch for each tuning.

    python scripts/sweep.py --config c2 --reps 200

Times back-to-back launches over rotating buffer pairs (> 3x L2) with CUDA
events; prints one JSON line per variant to stdout.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_1904_12380_b200 import _native, configs  # noqa: E402

K1_SHAPES = {
    # (vec, lpr, nv, u, pf) -- entries instantiated in sk_api.cu
    "c2": [(4, 8, 4, 1, 0), (4, 16, 2, 1, 0), (4, 8, 4, 2, 0), (4, 16, 2, 2, 0), (8, 8, 2, 1, 0)],
    "c5a": [(4, 16, 4, 1, 0), (4, 16, 4, 1, 1), (4, 16, 4, 2, 0), (4, 32, 2, 1, 0),
            (4, 32, 2, 2, 0), (8, 16, 2, 1, 0)],
    "c3": [(4, 32, 8, 1, 0), (4, 32, 8, 1, 1), (8, 32, 4, 1, 0)],
    "c1": [(1, 16, 4, 2, 0), (1, 16, 4, 1, 1), (1, 32, 2, 2, 0)],
}


def bench_once(x, ys, rows, cols, reps, stream):
    L = _native.lib()
    R = len(ys)
    flag = torch.full((1,), -1, dtype=torch.int64, device=x[0].device)

    def launch(i):
        _native.check(L.sk_softmax_f32(x[i % R].data_ptr(), ys[i % R].data_ptr(), rows, cols, cols,
                                       cols, 0, flag.data_ptr(), None, 0, stream.cuda_stream))

    with torch.cuda.stream(stream):
        for i in range(10):
            launch(i)
        g = torch.cuda.CUDAGraph()
        G = R * max(1, 32 // R)
        with torch.cuda.graph(g, stream=stream):
            for i in range(G):
                launch(i)
        g.replay()
        stream.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        n = max(1, reps // G)
        e0.record(stream)
        for _ in range(n):
            g.replay()
        e1.record(stream)
    stream.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (n * G)


def resident(record, xs, ys, rows, cols, args, s):
    """K3c vs K3g (group sizes x ring depths) vs split, on the same buffers."""
    _native.set_tuning("gres", 0)
    try:
        record("k3_cluster (gres off)", bench_once(xs, ys, rows, cols, args.reps, s))
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"variant": "k3_cluster", "error": str(e)}))
    _native.set_tuning("gres", 2)
    for gp in map(int, args.gres_ps.split(",")):
        for gs in map(int, args.gres_st.split(",")):
            _native.set_tuning("gres_p", gp)
            _native.set_tuning("gres_st", gs)
            try:
                record(f"k3_gres P={gp or 'auto'} st={gs or 'auto'}",
                       bench_once(xs, ys, rows, cols, args.reps, s))
            except Exception as e:  # noqa: BLE001
                print(json.dumps({"variant": f"gres {gp} st {gs}", "error": str(e)}))
    _native.set_tuning("gres_p", 0)
    _native.set_tuning("gres_st", 0)
    _native.set_tuning("gres", 1)
    _native.set_tuning("path", 2)
    record("split(k4)", bench_once(xs, ys, rows, cols, max(10, args.reps // 4), s))
    _native.set_tuning("path", -1)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c2")
    p.add_argument("--reps", type=int, default=200)
    p.add_argument("--grid-mults", default="1,2")
    p.add_argument("--shape", default="", help="RxC: synthetic N(0,4^2) matrix instead of a config")
    p.add_argument("--gres-ps", default="0,10,12,16,24,37,48,74",
                   help="K3g CTAs per row to try (0 = planner's choice)")
    p.add_argument("--gres-st", default="0", help="K3g ring depths to try (0 = planner's)")
    p.add_argument("--only-resident", action="store_true",
                   help="long rows: only the resident-row kernels (K3c / K3g) and split")
    args = p.parse_args()
    if args.shape:
        r, c = map(int, args.shape.lower().split("x"))
        spec = configs.InputSpec(f"shape{r}x{c}", r, c, "normal", 11, sigma=4.0)
    else:
        spec = configs.get(args.config)
    x_host = configs.generate(spec)
    dev = torch.device("cuda", 0)
    pair = 8 * spec.rows * spec.cols
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    R = max(2, -(-3 * l2 // pair))
    xs = [torch.from_numpy(x_host).to(dev)]
    xs += [xs[0].clone() for _ in range(R - 1)]
    ys = [torch.empty_like(xs[0]) for _ in range(R)]
    s = torch.cuda.Stream(dev)
    rows, cols = spec.rows, spec.cols
    out = []

    def record(tag, us):
        d = {"config": spec.name, "variant": tag, "us": us,
             "gbs": 8.0 * rows * cols / us / 1e3,
             "plan": _native.describe_plan(rows, cols, cols, cols, xs[0].data_ptr(),
                                           ys[0].data_ptr(), 0)}
        print(json.dumps(d), flush=True)
        out.append(d)

    record("default", bench_once(xs, ys, rows, cols, args.reps, s))
    if cols > 1024 and args.only_resident:
        resident(record, xs, ys, rows, cols, args, s)
    elif 1024 < cols <= 8192:
        for path in (2,):
            _native.set_tuning("path", path)
            record(f"path={path}", bench_once(xs, ys, rows, cols, args.reps, s))
        _native.set_tuning("path", -1)
    elif cols <= 1024:
        for path in (1, 2):  # K2 TMA block-per-row, K4 split, on the same rows
            _native.set_tuning("path", path)
            try:
                record(f"path={path}", bench_once(xs, ys, rows, cols, args.reps, s))
            except Exception as e:  # noqa: BLE001
                print(json.dumps({"variant": f"path={path}", "error": str(e)}))
        _native.set_tuning("path", -1)
        _native.set_tuning("pdl", 0)
        record("default pdl=0", bench_once(xs, ys, rows, cols, args.reps, s))
        _native.set_tuning("pdl", 1)
        for vw, lpr, nv, u, pf in K1_SHAPES.get(spec.name, []):
            _native.set_tuning("vec8", 1 if vw == 8 else 0)
            for gm in map(int, args.grid_mults.split(",")):
                _native.set_tuning("k1_lpr", lpr)
                _native.set_tuning("k1_nv", nv)
                _native.set_tuning("k1_u", u)
                _native.set_tuning("k1_pf", pf)
                _native.set_tuning("grid_mult", gm)
                try:
                    record(f"k1 vec={vw} lpr={lpr} nv={nv} u={u} pf={pf} gm={gm}",
                           bench_once(xs, ys, rows, cols, args.reps, s))
                except Exception as e:  # noqa: BLE001
                    print(json.dumps({"variant": f"{lpr},{nv},{u},{pf}", "error": str(e)}))
        _native.set_tuning("vec8", 1)
        _native.set_tuning("k1_lpr", 0)
        _native.set_tuning("k1_pf", -1)
        _native.set_tuning("grid_mult", 0)
    else:
        _native.set_tuning("pdl", 0)
        record("default pdl=0", bench_once(xs, ys, rows, cols, args.reps, s))
        _native.set_tuning("pdl", 1)
        resident(record, xs, ys, rows, cols, args, s)
        _native.set_tuning("k3_impl", 5)  # K3c variants
        for onex, tpb in ((1, 512), (0, 1024)):
            _native.set_tuning("cluster_onex", onex)
            _native.set_tuning("cluster_tpb", tpb)
            try:
                record(f"k3_cluster onex={onex} tpb={tpb}", bench_once(xs, ys, rows, cols, args.reps, s))
            except Exception as e:  # noqa: BLE001
                print(json.dumps({"variant": f"cluster onex={onex} tpb={tpb}", "error": str(e)}))
        _native.set_tuning("cluster_onex", 0)
        _native.set_tuning("cluster_tpb", 512)
        for csz in (16, 12, 10, 8):
            _native.set_tuning("cluster_size", csz)
            try:
                record(f"k3_cluster size {csz}", bench_once(xs, ys, rows, cols, args.reps, s))
            except Exception as e:  # noqa: BLE001
                print(json.dumps({"variant": f"cluster {csz}", "error": str(e)}))
        _native.set_tuning("cluster_size", 0)
        _native.set_tuning("k3_impl", 3)
    # our own streaming copy kernel of the same bytes, several grid sizes
    L = _native.lib()
    for blocks in (0, 592, 1184, 2368, 4736):
        def launch_copy(i, blocks=blocks):
            _native.check(L.sk_copy_f32(xs[i % R].data_ptr(), ys[i % R].data_ptr(), rows * cols,
                                        blocks, s.cuda_stream))
        with torch.cuda.stream(s):
            for i in range(10):
                launch_copy(i)
            g = torch.cuda.CUDAGraph()
            G = R * max(1, 32 // R)
            with torch.cuda.graph(g, stream=s):
                for i in range(G):
                    launch_copy(i)
            g.replay()
            s.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            n = max(1, args.reps // G)
            e0.record(s)
            for _ in range(n):
                g.replay()
            e1.record(s)
        s.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (n * G)
        print(json.dumps({"config": spec.name, "variant": f"sk_copy blocks={blocks}", "us": us,
                          "gbs": 8.0 * rows * cols / us / 1e3}), flush=True)
    # copy roofline in the same run: D2D copy of the same bytes (bound_probe analog)
    a = xs[0]
    b = ys[0]
    with torch.cuda.stream(s):
        for _ in range(5):
            b.copy_(a)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for i in range(50):
            ys[i % R].copy_(xs[i % R])
        e1.record(s)
    s.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 50
    print(json.dumps({"config": spec.name, "variant": "torch copy_ (same bytes)", "us": us,
                      "gbs": 8.0 * rows * cols / us / 1e3}), flush=True)


if __name__ == "__main__":
    main()
