// conv_prod0.cu -- instantiates the conv kernel for producer kind 0
// (TMA boxes); see conv_kernel.cuh.
#include "conv_kernel.cuh"

namespace wfb {
template const void* conv_kernel_fn<0>(int, wf_dtype, int);
}  // namespace wfb
