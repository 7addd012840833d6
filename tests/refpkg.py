"""The reference package (softmax_kit) as installed into baseline/_ref by
`pip install --no-deps --target baseline/_ref <copy of /root/reference/pkg>`
 -- the live reference for drop-in tests; None when absent."""

import os
import sys

from tests.conftest import ROOT

REF_DIR = ROOT / "baseline" / "_ref"


def load():
    if not (REF_DIR / "softmax_kit" / "kernels.py").exists():
        return None
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    os.environ.setdefault("NUMBA_CACHE_DIR", f"/tmp/sk_numba_{os.getuid()}")
    try:
        import softmax_kit.errors as errors
        import softmax_kit.kernels as kernels
        import softmax_kit.simd_reduce as simd_reduce
        import softmax_kit.tensor as tensor
    except Exception:  # noqa: BLE001
        return None

    class Ref:
        pass

    r = Ref()
    r.errors, r.kernels, r.tensor, r.simd_reduce = errors, kernels, tensor, simd_reduce
    return r
