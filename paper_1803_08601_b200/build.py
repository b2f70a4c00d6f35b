"""Build libspmm.so in-tree with nvcc for sm_100a (no torch in the library, no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libspmm.so")
SOURCES = [os.path.join(CSRC, "spmm_api.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("common.cuh", "ptx.cuh", "tile.cuh", "merge.cuh", "merge_w.cuh")] + \
    [os.path.join(ROOT, "include", "spmm.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xcompiler", "-fvisibility=hidden",
]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Build libspmm.so (or a variant at `out` with extra -D defines, for tuning experiments)."""
    lib = out or LIB
    if not force and out is None and not needs_build():
        return LIB
    cmd = [_nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-o", lib + ".tmp", *SOURCES]
    if verbose:
        cmd += ["-Xptxas", "-v"]
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    ap.add_argument("--out", default=None)
    ap.add_argument("-D", action="append", default=[])
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.v, out=a.out, defines=a.D))
