// inst_f32_plus_times.cu -- kernel instances for float values, plus-times semiring (one translation unit
// per kind so the library builds in parallel; see launch_kernels.cuh).
#include "launch_kernels.cuh"

namespace spmm {
SPMM_INSTANTIATE_KIND(float, SR_PLUS_TIMES)
}  // namespace spmm
