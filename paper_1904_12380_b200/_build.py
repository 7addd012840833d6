"""In-tree build of the native library (sm_100a) and, for tests, the C oracle.

The product library ``libsoftmax_b200.so`` is compiled straight with nvcc
(no torch extension machinery): the kernels are reached through the plain
C ABI in ``include/softmax_b200.h``.  The .so lands next to this file so it
travels with the repo snapshot to the GPU box (it is git-ignored, not
gpurun-ignored).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libsoftmax_b200.so"
ORACLE_DIR = ROOT / "oracle"
ORACLE_LIB = ORACLE_DIR / "libsk_oracle.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    *ARCH,
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "-Xcompiler",
    "-fPIC",
    "-Xcompiler",
    "-O3",
    # no --use_fast_math: expf must stay the accurate libdevice expf and 1/x the
    # IEEE reciprocal (kernels.py:171-189 numeric contract).
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found (need CUDA 12.9 toolkit)")


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))


def _deps() -> list[Path]:
    return (_sources() + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h"))
            + [ROOT / "include" / "softmax_b200.h"])


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_native(force: bool = False, verbose: bool = False) -> Path:
    """Compile every .cu/.cpp under csrc/ into libsoftmax_b200.so (sm_100a)."""
    if not force and not _stale(LIB, _deps()):
        return LIB
    nvcc = _nvcc()
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    objs = []
    procs = []
    for src in _sources():
        obj = objdir / (src.name + ".o")
        objs.append(obj)
        cmd = [nvcc, *NVCC_FLAGS, "-I", str(ROOT / "include"), "-c", str(src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{out.decode(errors='replace')}")
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-Xcompiler", "-fPIC", *map(str, objs), "-o", str(tmp),
           "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


TORCH_OPS_SRC = PKG / "torch_ops" / "sk_torch_ops.cpp"
TORCH_OPS_LIB = PKG / "libsoftmax_b200_torch.so"


def build_torch_ops(force: bool = False) -> Path:
    """torch.ops.softmax_b200.* (TORCH_LIBRARY launchers over the C ABI), g++
    against torch's headers, linked to libsoftmax_b200.so via $ORIGIN."""
    deps = [TORCH_OPS_SRC, ROOT / "include" / "softmax_b200.h", LIB]
    if not force and not _stale(TORCH_OPS_LIB, deps):
        return TORCH_OPS_LIB
    import torch
    from torch.utils import cpp_extension as ce

    inc = [str(Path(torch.__file__).parent / "include"),
           str(Path(torch.__file__).parent / "include" / "torch" / "csrc" / "api" / "include"),
           "/usr/local/cuda/include", str(ROOT / "include")]
    libdir = str(Path(torch.__file__).parent / "lib")
    abi = int(torch._C._GLIBCXX_USE_CXX11_ABI)
    tmp = TORCH_OPS_LIB.with_suffix(".so.tmp")
    cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", f"-D_GLIBCXX_USE_CXX11_ABI={abi}",
           *[f"-I{i}" for i in inc], str(TORCH_OPS_SRC), "-o", str(tmp),
           f"-L{libdir}", f"-L{PKG}", "-lsoftmax_b200", "-lc10", "-lc10_cuda", "-ltorch",
           "-ltorch_cpu", "-ltorch_cuda", "-Wl,-rpath,$ORIGIN", f"-Wl,-rpath,{libdir}",
           "-L/usr/local/cuda/lib64", "-lcudart"]
    del ce
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"torch ops build failed: {' '.join(cmd)}\n{r.stdout}{r.stderr}")
    os.replace(tmp, TORCH_OPS_LIB)
    return TORCH_OPS_LIB


def build_oracle(force: bool = False) -> Path:
    """Compile the C restatement of the reference (test infrastructure only;
    the recipe lives with the oracle, oracle/oracle.py:build)."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("_sk_oracle_build", ORACLE_DIR / "oracle.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.build(force)


REF_SRC = Path("/root/reference/pkg")
REF_DST = ROOT / "baseline" / "_ref"


def install_reference() -> Path | None:
    """Install the UNMODIFIED reference package into baseline/_ref (git-ignored,
    travels with the snapshot) when its sources are present and it is not there
    yet: the reference arm of bench.py and the live-reference tests use it.  The
    sources are read-only, so pip builds from a copy under /tmp."""
    if (REF_DST / "softmax_kit").is_dir():
        return REF_DST
    if not REF_SRC.is_dir():
        return None
    import tempfile

    with tempfile.TemporaryDirectory(prefix="sk_refpkg_") as tmp:
        src = Path(tmp) / "pkg"
        shutil.copytree(REF_SRC, src)
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
               "--no-deps", "--find-links", "/opt/wheelhouse", "--target", str(REF_DST), str(src)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            print(f"reference install failed (reference arm falls back to the C port):\n"
                  f"{r.stdout[-2000:]}{r.stderr[-2000:]}", file=sys.stderr)
            return None
    return REF_DST


if __name__ == "__main__":
    install_reference()
    build_native(force="--force" in sys.argv, verbose=True)
    build_torch_ops(force="--force" in sys.argv)
    build_oracle(force="--force" in sys.argv)
    print(LIB, ORACLE_LIB)
