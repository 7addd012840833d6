"""Golden vectors for the 1-D component operations, from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_components.py

Imports the reference from a temp copy (see make_golden.py) and records, for
a set of seeded rows, the outputs of row_max_scalar, subtract_broadcast,
value_clip, exp_batch, row_sum_scalar, scale_reciprocal and row_stats
(kernels.py:229-276) into golden_components.npz.  The GPU test
(tests/test_gpu_components.py) compares paper_1904_12380_b200.components
against these.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

from make_golden import _import_reference  # noqa: E402

LENGTHS = (1, 2, 7, 50, 128, 1000, 4097, 20000)
CLIP_SCALARS = np.array([0.0, -1.0, -63.9, -64.0, -64.1, -100.0, -1e30, 5.0], np.float32)


def rows():
    rng = np.random.default_rng(20261020)
    out = {}
    for C in LENGTHS:
        r = rng.uniform(-30.0, 30.0, C).astype(np.float32)
        if C >= 8:
            r[C // 2] = 60.0  # a dominant logit
            r[1] = -120.0     # far below the max
        out[f"u{C}"] = r
    out["spec_big"] = np.array([1000, 999, -1000], np.float32)
    out["spec_123"] = np.array([1, 2, 3], np.float32)
    return out


def main() -> None:
    K, _, _ = _import_reference()
    out: dict[str, np.ndarray] = {"clip/x": CLIP_SCALARS,
                                  "clip/y": np.array([K.value_clip(v) for v in CLIP_SCALARS],
                                                     np.float32)}
    for name, r in rows().items():
        out[f"{name}/row"] = r
        m = K.row_max_scalar(r)
        out[f"{name}/max"] = np.array([m], np.float32)
        sh = K.subtract_broadcast(r, m)
        out[f"{name}/sub_max"] = sh
        out[f"{name}/sub_325"] = K.subtract_broadcast(r, 3.25)
        e = K.exp_batch(sh.copy())
        out[f"{name}/exp"] = e
        s = K.row_sum_scalar(e)
        out[f"{name}/sum_exp"] = np.array([s], np.float32)
        out[f"{name}/sum_row"] = np.array([K.row_sum_scalar(r)], np.float32)
        out[f"{name}/scaled"] = K.scale_reciprocal(e, s)
        st = K.row_stats(r)
        out[f"{name}/stats"] = np.array([st.max, st.sum], np.float32)
    np.savez_compressed(HERE / "golden_components.npz", **out)
    print("wrote", HERE / "golden_components.npz", len(out), "arrays")


if __name__ == "__main__":
    main()
