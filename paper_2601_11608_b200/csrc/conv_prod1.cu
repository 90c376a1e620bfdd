// conv_prod1.cu -- instantiates the conv kernel for producer kind 1
// (row gather, folded layout); see conv_kernel.cuh.
#include "conv_kernel.cuh"

namespace wfb {
template const void* conv_kernel_fn<1>(int, wf_dtype, int);
}  // namespace wfb
