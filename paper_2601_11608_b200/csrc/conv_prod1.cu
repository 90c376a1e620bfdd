// conv_prod1.cu -- instantiates the conv kernel for producer kind 1
// (software gather, folded layout); see conv_kernel.cuh.
#include "conv_kernel.cuh"

namespace wfb {
template cudaError_t launch_conv_prod<1>(const ConvArgs&, const TmaMaps&, int, int, cudaStream_t, int, wf_dtype, int);
}  // namespace wfb
