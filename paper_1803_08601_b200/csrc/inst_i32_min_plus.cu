// inst_i32_min_plus.cu -- kernel instances for int values, min-plus semiring (one translation unit
// per kind so the library builds in parallel; see launch_kernels.cuh).
#include "launch_kernels.cuh"

namespace spmm {
SPMM_INSTANTIATE_KIND(int, SR_MIN_PLUS)
}  // namespace spmm
