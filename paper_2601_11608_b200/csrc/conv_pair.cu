// conv_pair.cu -- instantiates the CTA-pair (cta_group::2) conv kernel; see conv_kernel.cuh.
#include "conv_kernel.cuh"

namespace wfb {

cudaError_t launch_conv_pair(const ConvArgs& args, const TmaMaps& maps, int grid, int smem, cudaStream_t st,
                             wf_dtype out, int ch) {
  if (ch == 64) {
    if (out == WF_BF16) return launch_pair_typed<__nv_bfloat16, 64>(args, maps, grid, smem, st);
    if (out == WF_F16) return launch_pair_typed<__half, 64>(args, maps, grid, smem, st);
    return launch_pair_typed<float, 64>(args, maps, grid, smem, st);
  }
  if (out == WF_BF16) return launch_pair_typed<__nv_bfloat16, 32>(args, maps, grid, smem, st);
  if (out == WF_F16) return launch_pair_typed<__half, 32>(args, maps, grid, smem, st);
  return launch_pair_typed<float, 32>(args, maps, grid, smem, st);
}

cudaError_t launch_conv_mc(const ConvArgs& args, const TmaMaps& maps, int grid, int smem, cudaStream_t st,
                           wf_dtype out, int ch) {
  if (ch == 64) {
    if (out == WF_BF16) return launch_mc_typed<__nv_bfloat16, 64>(args, maps, grid, smem, st);
    if (out == WF_F16) return launch_mc_typed<__half, 64>(args, maps, grid, smem, st);
    return launch_mc_typed<float, 64>(args, maps, grid, smem, st);
  }
  if (out == WF_BF16) return launch_mc_typed<__nv_bfloat16, 32>(args, maps, grid, smem, st);
  if (out == WF_F16) return launch_mc_typed<__half, 32>(args, maps, grid, smem, st);
  return launch_mc_typed<float, 32>(args, maps, grid, smem, st);
}

}  // namespace wfb
