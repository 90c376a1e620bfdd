// conv_prod4.cu -- instantiates the conv kernel for producer kind 4 (direct
// gather of unaligned rows from global memory, folded layout); see conv_kernel.cuh.
#include "conv_kernel.cuh"

namespace wfb {
template const void* conv_kernel_fn<4>(int, wf_dtype, int);
}  // namespace wfb
