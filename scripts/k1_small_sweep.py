"""Short rows at 64 MiB: every K1 instantiation that covers C (default plan first), grid multiplier 0 / 2."""
import json, sys
from pathlib import Path
ROOT = Path("/root/repo") if Path("/root/repo/scripts").exists() else Path(".")
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "scripts"))
import torch
from paper_1904_12380_b200 import _native, configs
from sweep import bench_once
TABLE4 = [(4,4,1,4,0),(4,8,1,4,0),(4,16,1,4,0),(4,8,2,2,0),(4,8,4,1,0),(4,8,4,2,0),(4,16,2,2,0),(4,16,2,1,0),(4,16,4,1,0),(4,16,4,2,0),(4,32,1,4,0),(4,32,2,2,0),(4,32,4,1,0),(4,32,1,2,0),(4,32,2,1,0),(4,8,4,1,1),(4,16,2,1,1),(4,16,4,1,1),(4,32,2,1,1),(4,16,1,4,1),(4,8,1,4,1),(4,4,1,8,0),(4,8,1,8,0),(4,16,1,8,0),(4,16,1,8,1)]
TABLE1 = [(1,8,1,4,0),(1,16,1,4,0),(1,32,1,4,0),(1,16,4,2,0),(1,32,2,2,0),(1,32,4,1,0),(1,16,4,2,1),(1,16,4,1,1),(1,16,4,4,0),(1,16,4,4,1),(1,16,4,8,0)]
s = torch.cuda.Stream()
ROWS = int(sys.argv[2]) if len(sys.argv) > 2 else 0  # 0: a 64 MiB job
for C in map(int, sys.argv[1].split(",")):
    rows = ROWS or (16 << 20) // C
    spec = configs.InputSpec(f"len{C}", rows, C, "normal", 7, sigma=4.0)
    x0 = torch.from_numpy(configs.generate(spec)).cuda()
    R = max(6, -(-3 * (126 << 20) // (8 * rows * C)))
    xs = [x0] + [x0.clone() for _ in range(R - 1)]
    ys = [torch.empty_like(x0) for _ in range(R)]
    tab = TABLE4 if C % 4 == 0 else TABLE1
    for shp in [None] + tab:
        if shp is not None:
            vec, lpr, nv, u, pf = shp
            if lpr * nv * vec < C or lpr * nv * vec >= 4 * C and lpr > 4: continue
            for k, v in (("k1_lpr", lpr), ("k1_nv", nv), ("k1_u", u), ("k1_pf", pf)): _native.set_tuning(k, v)
        for gm in (0, 2):
            _native.set_tuning("grid_mult", gm)
            try:
                us = bench_once(xs, ys, rows, C, 100, s)
                print(json.dumps({"C": C, "rows": rows, "plan": _native.describe_plan(rows, C), "gm": gm, "us": round(us, 2), "gbs": round(8 * rows * C / us / 1e3)}), flush=True)
            except Exception as e:
                print(json.dumps({"C": C, "shape": shp, "err": str(e)}), flush=True)
        for k, v in (("k1_lpr", 0), ("k1_nv", 0), ("k1_u", 0), ("k1_pf", -1), ("grid_mult", 0)): _native.set_tuning(k, v)
