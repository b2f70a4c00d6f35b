"""Build libspmm.so in-tree with nvcc for sm_100a (no torch in the library, no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libspmm.so")
# the C ABI / planner, and one kernel-instance translation unit per value type x semiring (compiled in
# parallel, then linked into one shared library)
SOURCES = [os.path.join(CSRC, f) for f in ("spmm_api.cu", "inst_f32_plus_times.cu", "inst_f32_min_plus.cu",
                                           "inst_i32_plus_times.cu", "inst_i32_min_plus.cu", "csr_split.cu")]
DEPS = SOURCES + sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))) + \
    [os.path.join(ROOT, "include", "spmm.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xcompiler", "-fvisibility=hidden",
]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def source_sha16(defines=()) -> str:
    """Identity of a build from its inputs: sha256 over every source / header the library is built from,
    the nvcc flags and extra defines.  (The .so itself is not bit-reproducible: nvcc names internal-
    linkage device symbols after the compiling process, so two builds of the same sources differ in a
    few symbol-name bytes while their SASS is identical.)"""
    import hashlib
    h = hashlib.sha256()
    for d in sorted(DEPS):
        h.update(os.path.relpath(d, ROOT).encode())
        with open(d, "rb") as f:
            h.update(f.read())
    h.update(" ".join(NVCC_FLAGS + [f"-D{d}" for d in defines]).encode())
    return h.hexdigest()[:16]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Build libspmm.so (or a variant at `out` with extra -D defines, for tuning experiments): every
    translation unit is compiled to an object in parallel, then linked with nvcc -shared."""
    from concurrent.futures import ThreadPoolExecutor
    import hashlib
    lib = out or LIB
    if not force and out is None and not needs_build():
        return LIB
    tag = hashlib.sha1(("|".join(defines) + "|" + lib).encode()).hexdigest()[:10]
    odir = os.path.join(ROOT, "build", "obj_" + tag)
    os.makedirs(odir, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]
    extra = ["-Xptxas", "-v"] if verbose else []

    def compile_one(src):
        obj = os.path.join(odir, os.path.basename(src)[:-3] + ".o")
        cmd = [_nvcc(), *NVCC_FLAGS, *dflags, *extra, "-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
        return obj

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    subprocess.check_call([_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib + ".tmp", *objs])
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
