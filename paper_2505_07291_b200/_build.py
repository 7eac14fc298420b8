"""Build the sm_100a shared library in-tree (``nvcc``, no JIT cache).

``python -m paper_2505_07291_b200._build`` or ``__graft_entry__.build()``.
Output: ``paper_2505_07291_b200/_lib/libtoploc_b200.so`` (git-ignored; travels to
the GPU box with the gpurun snapshot).
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC = os.path.join(PKG, "csrc", "toploc_b200.cu")
OUT_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(OUT_DIR, "libtoploc_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xptxas", "-v",
    "-Xcompiler", "-fPIC", "-shared",
    "--expt-relaxed-constexpr",
]


def _deps():
    d = os.path.join(PKG, "csrc")
    return [os.path.join(d, f) for f in os.listdir(d)] + [os.path.join(ROOT, "include", "toploc_b200.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in _deps())


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    lib = out or LIB
    if not force and out is None and not needs_build():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    tmp = lib + ".tmp"
    cmd = [NVCC, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-o", tmp, SRC, "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr}")
    if verbose:
        sys.stderr.write(res.stderr)
    with open(lib + ".ptxas.log" if out else os.path.join(OUT_DIR, "ptxas.log"), "w") as f:
        f.write(res.stderr)
    os.replace(tmp, lib)
    return lib


CHECKED_LIB = os.path.join(OUT_DIR, "libtoploc_b200_checked.so")


def build_checked(force: bool = False) -> str:
    """The -DTL_CHECKED=1 library: device asserts on the index, workspace and chunk-geometry
    arithmetic (tests/test_gpu_checked.py runs the GPU fuzz suites against it; select it with
    TOPLOC_B200_LIB)."""
    if not force and os.path.exists(CHECKED_LIB) and os.path.getmtime(CHECKED_LIB) >= max(
            os.path.getmtime(f) for f in _deps()):
        return CHECKED_LIB
    return build(force=True, out=CHECKED_LIB, defines=("TL_CHECKED=1",))


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
