// conv_prod2.cu -- instantiates the conv kernel for producer kind 2
// (row gather, explicit im2col); see conv_kernel.cuh.
#include "conv_kernel.cuh"

namespace wfb {
template const void* conv_kernel_fn<2>(int, wf_dtype, int);
}  // namespace wfb
