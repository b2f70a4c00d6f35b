"""paper_1803_08601_b200 -- B200-native (sm_100a) CSR SpMM hot path of Yang, Buluc, Owens,
"Design Principles for Sparse Matrix Multiplication on the GPU" (arXiv 1803.08601).

  csrc/        CUDA kernels (row split §4.1, merge-based Alg. 1 §4.2) + the C ABI of include/spmm.h
  spmm.py      ctypes binding with the C names + CsrSpmm convenience class (torch = memory/streams only)
  dist.py      multi-GPU row-block partition + NCCL broadcast of B (north_star)
  synth.py     seeded synthetic inputs (no method arithmetic; shared with the oracle tests)
  build.py     nvcc build of libspmm.so for sm_100a
"""

__all__ = ["spmm", "synth", "build", "dist"]
