// conv_prod2.cu -- instantiates the conv kernel for producer kind 2
// (software gather, explicit im2col); see conv_kernel.cuh.
#include "conv_kernel.cuh"

namespace wfb {
template cudaError_t launch_conv_prod<2>(const ConvArgs&, const TmaMaps&, int, int, cudaStream_t, int, wf_dtype, int);
}  // namespace wfb
