"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It copies /root/reference/pkg/src/softmax_kit to a temp dir (numba's
cache=True would otherwise write into the read-only reference tree), imports
it with NUMBA_CACHE_DIR pointed at the temp dir, and records:

* golden.npz  -- small input/output vectors: SPEC known answers, a sweep of
  row lengths (incl. clip-triggering logits) through every ladder rung,
  rows of the c1/c3 configs, fill_uniform prefixes, lane max/sum results;
* golden.json -- SHA-256 of full-size reference fill_uniform streams and of
  the reference ReferenceClipped output on the full BASELINE configs (the
  inputs come from this repo's generators; their hashes are recorded too).

The reference cannot travel to the GPU box; these committed fixtures are how
the oracle (oracle/sk_oracle.c) and the CUDA path are pinned to it.
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
REF_SRC = Path("/root/reference/pkg/src/softmax_kit")


def _import_reference():
    tmp = Path(tempfile.mkdtemp(prefix="skref_"))
    shutil.copytree(REF_SRC, tmp / "softmax_kit")
    os.environ["NUMBA_CACHE_DIR"] = str(tmp / "numba_cache")
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(tmp))
    import softmax_kit.kernels as K  # noqa: E402
    import softmax_kit.simd_reduce as S  # noqa: E402
    import softmax_kit.tensor as T  # noqa: E402

    return K, S, T


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8).reshape(-1).data).hexdigest()


def main(full: bool = True) -> None:
    K, S, T = _import_reference()
    sys.path.insert(0, str(ROOT))
    from paper_1904_12380_b200 import configs

    V = K.KernelVariant
    rungs = {
        "clipped": V.REFERENCE_CLIPPED,
        "inference": V.REFERENCE_INFERENCE,
        "mkl": V.MKL_STYLE_SCALAR,
        "vecsum": V.VECTORIZED_SUM,
        "fullvec": V.FULL_VECTORIZED,
        "approx": V.FULL_VECTORIZED_APPROX_EXP,
    }

    def ref_softmax(x2d: np.ndarray, variant) -> np.ndarray:
        m = T.alloc_matrix(*x2d.shape)
        m.view2d[...] = x2d
        return K.softmax(m, variant).view2d.copy()

    out: dict[str, np.ndarray] = {}
    meta: dict = {"reference": str(REF_SRC), "numpy": np.__version__}

    # --- SPEC known answers
    spec_cases = {
        "spec_123": np.array([[1, 2, 3]], np.float32),
        "spec_zeros": np.zeros((1, 4), np.float32),
        "spec_single": np.array([[7.5]], np.float32),
        "spec_big": np.array([[1000, 999, -1000]], np.float32),
        "spec_clip": np.array([[0.0, -100.0, -63.9, -64.0, -64.1, -87.5, -200.0, 5.0]], np.float32),
    }
    for name, x in spec_cases.items():
        out[f"{name}/x"] = x
        for r in ("clipped", "inference"):
            out[f"{name}/{r}"] = ref_softmax(x, rungs[r])

    # --- row-length sweep through every rung (ragged/odd/aligned C)
    sweep = [1, 2, 3, 4, 5, 7, 8, 16, 31, 32, 33, 49, 50, 51, 63, 64, 65, 100, 127, 128, 129,
             255, 256, 257, 511, 1000, 1023, 1024, 1025, 2048, 4097, 8192, 8193]
    meta["sweep"] = sweep
    for C in sweep:
        R = 5 if C <= 256 else (2 if C <= 1025 else 1)
        m = T.alloc_matrix(R, C)
        T.fill_uniform(m, T.FillSpec(seed=1000 + C, low=-20.0, high=20.0))
        x = m.view2d.copy()
        if C >= 4:  # make the clip fire: far-below-max logits
            x[0, C // 3] = -150.0
            x[-1, C - 1] = -90.0
        if C >= 8:
            x[R // 2, 1] = 40.0  # a dominant logit
        out[f"sweep/{C}/x"] = x
        for r in ("clipped", "inference", "approx"):
            out[f"sweep/{C}/{r}"] = ref_softmax(x, rungs[r])

    # --- c1 rows and c3 rows (inputs from this repo's generators)
    c1 = configs.generate("c1")
    out["c1/x"] = c1[:64].copy()
    out["c1/clipped"] = ref_softmax(c1[:64], rungs["clipped"])
    c3 = configs.generate("c3")
    rows3 = np.unique(np.nonzero(c3 == -100.0)[0])[:32]
    out["c3/rows"] = rows3.astype(np.int64)
    out["c3/x"] = c3[rows3].copy()
    out["c3/clipped"] = ref_softmax(c3[rows3], rungs["clipped"])

    # --- fill_uniform (tensor.py:106-121) prefixes and full-stream hashes
    fills = [(1, -10.0, 10.0, 65536 * 128), (42, -5.0, 5.0, 128 * 1000), (7, -0.5, 3.25, 4099)]
    meta["fill_uniform"] = []
    for seed, lo, hi, n in fills:
        m = T.alloc_matrix(1, n)
        T.fill_uniform(m, T.FillSpec(seed=seed, low=lo, high=hi))
        out[f"fill/{seed}/prefix"] = m.data[:64].copy()
        meta["fill_uniform"].append({"seed": seed, "low": lo, "high": hi, "n": n,
                                     "sha256": sha(m.data)})

    # --- lane reductions (simd_reduce.py:149-209)
    rng = np.random.default_rng(123)
    for W in (4, 8, 16):
        for n in (1, 3, 7, 11, 64, 515):
            a = rng.uniform(-10, 10, n).astype(np.float32)
            out[f"lanes/{W}/{n}/a"] = a
            out[f"lanes/{W}/{n}/max"] = np.array([S.vmax(a, S.LaneConfig(W))], np.float32)
            out[f"lanes/{W}/{n}/sum"] = np.array([S.vsum(a, S.LaneConfig(W))], np.float32)

    # --- full-size ReferenceClipped output hashes on the BASELINE configs
    meta["configs"] = {}
    names = ["c1", "c2", "c3", "c4", "c5a", "c5b"] if full else ["c1", "c2", "c3"]
    for name in names:
        spec = configs.get(name)
        x = configs.generate(spec)
        m = T.alloc_matrix(spec.rows, spec.cols)
        m.view2d[...] = x
        y = K.softmax(m, V.REFERENCE_CLIPPED)
        meta["configs"][name] = {
            "shape": [spec.rows, spec.cols],
            "input_sha256": sha(x),
            "ref_clipped_sha256": sha(y.data),
            "row0_sum": float(np.sum(y.view2d[0], dtype=np.float64)),
            "min": float(y.data.min()),
            "max": float(y.data.max()),
        }
        print(name, meta["configs"][name], flush=True)
        del x, m, y

    np.savez_compressed(HERE / "golden.npz", **out)
    (HERE / "golden.json").write_text(json.dumps(meta, indent=1) + "\n")
    print("wrote", HERE / "golden.npz", HERE / "golden.json")


if __name__ == "__main__":
    main(full="--small" not in sys.argv)
