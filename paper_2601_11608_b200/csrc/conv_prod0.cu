// conv_prod0.cu -- instantiates the conv kernel for producer kind 0
// (TMA boxes); see conv_kernel.cuh.
#include "conv_kernel.cuh"

namespace wfb {
template cudaError_t launch_conv_prod<0>(const ConvArgs&, const TmaMaps&, int, int, cudaStream_t, int, wf_dtype, int);
}  // namespace wfb
