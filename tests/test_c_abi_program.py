"""The boundary used from plain C (no Python, no torch): tests/c/abi_smoke.c includes only
include/spmm.h and cuda_runtime.h and links libspmm.so.  -m "not gpu": it compiles and links as C11
(the header is valid C).  -m gpu: it runs C = P*B for a permutation matrix with an empty row through
AUTO / ROWSPLIT / MERGE in fp32 plus-times and int32 min-plus and checks every element bit-exactly
against the closed form (SURVEY.md §8(c) pins)."""
import os
import subprocess

import pytest

from paper_1803_08601_b200 import build as spmm_build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _compile(tmp_path):
    lib = spmm_build.build()
    libdir = os.path.dirname(lib)
    exe = str(tmp_path / "abi_smoke")
    cmd = ["gcc", "-std=c11", "-Wall", "-Werror", "-O2", f"-I{ROOT}/include", f"-I{CUDA}/include",
           os.path.join(ROOT, "tests", "c", "abi_smoke.c"), "-o", exe, f"-L{libdir}", "-l:libspmm.so",
           f"-L{CUDA}/lib64", "-lcudart", f"-Wl,-rpath,{libdir}:{CUDA}/lib64"]
    subprocess.check_call(cmd)
    return exe


def test_c_program_compiles_against_header(tmp_path):
    assert os.path.exists(_compile(tmp_path))


@pytest.mark.gpu
def test_c_program_runs_on_gpu(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = _compile(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "abi_smoke ok" in r.stdout
