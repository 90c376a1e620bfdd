// conv_pair.cu -- instantiates the cluster kernels: CTA pairs (cta_group::2)
// and the multicast N-tile cluster; see conv_kernel.cuh.
#include "conv_kernel.cuh"

namespace wfb {

const void* conv_kernel_fn_pair(wf_dtype out, int ch) {
  if (ch == 64) {
    if (out == WF_BF16) return kernel_ptr<0, __nv_bfloat16, 64, 0, 2>();
    if (out == WF_F16) return kernel_ptr<0, __half, 64, 0, 2>();
    return kernel_ptr<0, float, 64, 0, 2>();
  }
  if (out == WF_BF16) return kernel_ptr<0, __nv_bfloat16, 32, 0, 2>();
  if (out == WF_F16) return kernel_ptr<0, __half, 32, 0, 2>();
  return kernel_ptr<0, float, 32, 0, 2>();
}

const void* conv_kernel_fn_mc(wf_dtype out, int ch) {
  if (ch == 64) {
    if (out == WF_BF16) return kernel_ptr<0, __nv_bfloat16, 64, 0, 1, 1>();
    if (out == WF_F16) return kernel_ptr<0, __half, 64, 0, 1, 1>();
    return kernel_ptr<0, float, 64, 0, 1, 1>();
  }
  if (out == WF_BF16) return kernel_ptr<0, __nv_bfloat16, 32, 0, 1, 1>();
  if (out == WF_F16) return kernel_ptr<0, __half, 32, 0, 1, 1>();
  return kernel_ptr<0, float, 32, 0, 1, 1>();
}

const void* conv_kernel_fn_mc5(wf_dtype out) {
  if (out == WF_BF16) return kernel_ptr<0, __nv_bfloat16, 32, 5, 1, 1>();
  if (out == WF_F16) return kernel_ptr<0, __half, 32, 5, 1, 1>();
  return kernel_ptr<0, float, 32, 5, 1, 1>();
}

}  // namespace wfb
