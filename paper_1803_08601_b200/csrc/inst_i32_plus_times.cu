// inst_i32_plus_times.cu -- kernel instances for int values, plus-times semiring (one translation unit
// per kind so the library builds in parallel; see launch_kernels.cuh).
#include "launch_kernels.cuh"

namespace spmm {
SPMM_INSTANTIATE_KIND(int, SR_PLUS_TIMES)
}  // namespace spmm
