#!/usr/bin/env python
"""Small shapes through every kernel path, for compute-sanitizer.

    compute-sanitizer --tool memcheck python scripts/sanitize_target.py
Exits 1 if any output misses the oracle, so a sanitizer-clean run is also a
correct one.
"""

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1904_12380_b200 as sk  # noqa: E402
from paper_1904_12380_b200 import _native, phases, sharding, tensor  # noqa: E402

fails = 0


def run(x, mode=0, off=0, ld=None):
    global fails
    rows, cols = x.shape
    ld = ld or cols
    buf = torch.zeros(off + rows * ld + 4, device="cuda")
    xd = buf[off:off + rows * ld].view(rows, ld)[:, :cols]
    xd.copy_(torch.from_numpy(x))
    y = torch.empty(rows, cols, device="cuda")
    flag = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    _native.check(_native.lib().sk_softmax_f32(xd.data_ptr(), y.data_ptr(), rows, cols, ld, cols,
                                               mode, flag.data_ptr(), None, 0,
                                               torch.cuda.current_stream().cuda_stream))
    d = oracle.parity(y.cpu().numpy(), oracle.softmax_ref(x, mode == 0), approx=mode == 2)
    if not d["ok"]:
        fails += 1
        print("FAIL", x.shape, mode, off, ld, _native.describe_plan(rows, cols), d)


for C in (1, 3, 50, 128, 129, 1000, 1025, 2048, 3072, 4097, 6001, 8192, 8200, 20000, 65537):
    rows = 3 if C > 4096 else 9
    x = np.empty((rows, C), np.float32)
    tensor.fill_normal_array(x, C, 5.0)
    for mode in (0, 1, 2):
        run(x, mode)
    run(x, 0, off=1)
    run(x, 0, ld=C + 5)
x = np.empty((4, 30000), np.float32)
tensor.fill_normal_array(x, 7, 5.0)
for impl in (3, 5):  # K3g, K3c
    _native.set_tuning("k3_impl", impl)
    run(x)
_native.set_tuning("k3_impl", 3)
_native.set_tuning("path", 2)
run(x)
_native.set_tuning("path", -1)
# phases, row stats, host path
xd = torch.from_numpy(x).cuda()
p = phases.variant_pipeline(sk.KernelVariant.REFERENCE_CLIPPED, *x.shape)
b = torch.empty_like(xd)
p.maxsub(xd, b)
p.exp(b)
p.sumscale(b)
ops = sharding.cuda_column_ops()
m, s = ops.local_stats(xd, 0)
y = ops.normalize(xd, m, ops.rescale(m, m, s), 0)
h = sk.softmax(sk.Matrix2D.from_array(x), sk.KernelVariant.REFERENCE_CLIPPED)
if not oracle.parity(h.view2d, oracle.softmax_ref(x))["ok"]:
    fails += 1
torch.cuda.synchronize()
print("sanitize target done, fails =", fails)
sys.exit(1 if fails else 0)
