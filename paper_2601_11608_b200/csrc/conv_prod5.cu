// conv_prod5.cu -- instantiates the conv kernel for producer kind 5 (gather warps
// re-pitch stage units into an L2 ring, TMA boxes load the A stages from it);
// see conv_kernel.cuh.
#include "conv_kernel.cuh"

namespace wfb {
template const void* conv_kernel_fn<5>(int, wf_dtype, int);
}  // namespace wfb
