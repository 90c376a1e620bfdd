// kernels.hpp -- host-side launchers of the sm_100a kernels (internal).
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "plan.hpp"

namespace wfb {

// K1: expand + pack the filter into the tcgen05 B-operand layout, write the
// schedule table in front of it, and replicate the bias (fold.cpp:185-226).
wf_status launch_pack(const Schedule& S, const wf_conv_desc& d, const void* w, const float* b,
                      void* packed, float* b_rep, cudaStream_t st, std::string* err);

// Dense generalized expansion W'(KH,KW',f*C,r*Cout), fp32.
wf_status launch_expand_dense(const wf_conv_desc& d, int64_t f, const float* w, float* out,
                              cudaStream_t st, std::string* err);

// Prepared launches of one schedule (kernel arguments + encoded tensor maps
// per buffer set), most recent first. Repeated calls on the same buffers skip
// argument building and tensor-map encoding entirely.
struct PreparedLaunch;  // conv_fold.cu
struct LaunchCache {
  static constexpr size_t kMax = 8;
  std::mutex mu;
  std::vector<std::shared_ptr<const PreparedLaunch>> entries;
};

// K2: the folded implicit-GEMM convolution (TMA -> tcgen05.mma -> TMEM -> epilogue).
// num_sms <= 0: the device's SM count. cache may be null (no reuse).
wf_status launch_conv(const Schedule& S, const wf_conv_desc& d, const void* x, const void* workspace,
                      const void* packed, const float* b_rep, void* y, wf_dtype out_dtype, uint32_t epilogue,
                      cudaStream_t st, int num_sms, LaunchCache* cache, std::string* err);
int sm_count(int device);
// The re-pitch pass of a producer-3 schedule on its own (wf_repitch_input).
wf_status launch_repitch_input(const Schedule& S, const wf_conv_desc& d, const void* x, void* workspace,
                               cudaStream_t st, std::string* err);

// Every launch that writes a conv operand the kernel reads before its
// griddepcontrol.wait (the packed filter, the replicated bias) bumps this
// process-wide epoch; the next conv launch after a bump is made without the
// programmatic-dependent-launch attribute, so it cannot overlap that write.
void note_operand_write();
uint64_t operand_epoch();

// Exact-order fp32 direct conv (reference conv2d semantics, with padding).
// groups > 1: grouped conv of a block-diagonal dense filter (diagonal blocks only).
wf_status launch_conv_direct(const wf_conv_desc& d, const float* x, const float* w, float* y, int groups,
                             cudaStream_t st, std::string* err);
wf_status launch_cast_f32(const float* x, void* y, long long n, wf_dtype to, cudaStream_t st, std::string* err);
wf_status launch_bias_add(const float* y, const float* b, float* out, long long n, int C, int relu, cudaStream_t st,
                          std::string* err);
wf_status launch_blockdiag_check(const float* wd, int KH, int KW, int Cif, int Cof, int groups,
                                 unsigned long long* scratch, long long* first_bad, cudaStream_t st, std::string* err);
// Device fold for unaligned rows: copy x (rows of rb_in bytes) into ws (rows of rb_out, zero tail);
// planes > 0: each workspace row as `planes` core-column planes [q][folded col][16 B].
wf_status launch_repitch(const void* x, void* ws, long long rows, int rb_in, int rb_out, int planes,
                         cudaStream_t st, std::string* err);
wf_status launch_replicate_bias(const float* b, int cout, int r, float* out, cudaStream_t st, std::string* err);

}  // namespace wfb
