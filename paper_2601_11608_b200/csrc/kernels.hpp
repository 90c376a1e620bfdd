// kernels.hpp -- host-side launchers of the sm_100a kernels (internal).
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "plan.hpp"

namespace wfb {

// K1: expand + pack the filter into the tcgen05 B-operand layout, write the
// schedule table in front of it, and replicate the bias (fold.cpp:185-226).
wf_status launch_pack(const Schedule& S, const wf_conv_desc& d, const void* w, const float* b,
                      void* packed, float* b_rep, cudaStream_t st, std::string* err);

// Dense generalized expansion W'(KH,KW',f*C,r*Cout), fp32.
wf_status launch_expand_dense(const wf_conv_desc& d, int64_t f, const float* w, float* out,
                              cudaStream_t st, std::string* err);

// K2: the folded implicit-GEMM convolution (TMA -> tcgen05.mma -> TMEM -> epilogue).
wf_status launch_conv(const Schedule& S, const wf_conv_desc& d, const void* x, const void* packed,
                      const float* b_rep, void* y, wf_dtype out_dtype, uint32_t epilogue,
                      cudaStream_t st, int num_sms, std::string* err);

}  // namespace wfb
