// widthfold.hpp -- C++ host API of widthfold-b200.
//
// The reference operator interface lives at the reference's own include paths
// (include/widthfold/{errors,tensor,refconv,fold,blockdiag}.hpp): DenseTensor
// values in, DenseTensor values out, each operation running on the B200
// through the C-ABI (include/widthfold_b200.h). This header adds the device
// API under it: caller-owned device pointers (no allocation), a caller-given
// cudaStream_t, no host fallback -- the generalized device fold plan and the
// folded tcgen05 convolution with its once-per-weights packed filter.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "widthfold/blockdiag.hpp"
#include "widthfold/errors.hpp"
#include "widthfold/fold.hpp"
#include "widthfold/refconv.hpp"
#include "widthfold/tensor.hpp"
#include "widthfold_b200.h"

namespace widthfold {

// Turns a wf_status into the matching exception (message from wf_last_error).
void throw_on(wf_status st);

enum class Dtype { F32 = WF_F32, TF32 = WF_TF32, BF16 = WF_BF16, F16 = WF_F16 };

// Generalized device fold: KW > 1, stride, padding.
// factor == 0 picks the factor; returns the raw device schedule too.
struct DevicePlan {
  FoldPlan plan;
  wf_fold_plan raw{};
};
DevicePlan plan_device_fold(const ConvSpec& spec, std::int64_t factor, std::int64_t group_size, Dtype in_dtype);

// ---- device operations ------------------------------------------------------------
// Exact-order fp32 conv2d + optional bias/ReLU (reference conv2d/bias_add bits).
void conv2d_exact(const float* x, const float* w, float* y, const ConvSpec& spec, void* stream);
// Grouped exact-order conv of a block-diagonal dense filter (grouped_conv's engine).
void conv2d_grouped(const float* x, const float* w_dense, float* y, const ConvSpec& spec, std::int64_t groups,
                    void* stream);
void bias_add(const float* y, const float* b, float* out, std::int64_t n, std::int64_t c, bool relu, void* stream);
// y = (bf16 | f16) x on the device (round to nearest even)
void cast_f32(const float* x, void* y, std::int64_t n, Dtype to, void* stream);
void replicate_bias(const float* b, std::int64_t cout, std::int64_t factor, float* out, void* stream);
// Reference expand_filter_general (KW must be 1 -> IllegalFold), fp32 device.
void expand_filter_general(const float* w, const Shape& filter_shape, std::int64_t factor, float* out, void* stream);
// Generalized dense expansion (KH, KW', f*C, r*Cout).
void expand_filter_folded(const float* w, const Shape& filter_shape, std::int64_t factor, std::int64_t stride_w,
                          std::int64_t pad_w, float* out, void* stream);
Shape folded_filter_shape(const Shape& filter_shape, std::int64_t factor, std::int64_t stride_w, std::int64_t pad_w);
// Strict-zero check; throws NotBlockDiagonal. scratch: 8 bytes of device memory.
void check_block_diagonal(const float* w_dense, const Shape& dense_shape, std::int64_t groups, void* scratch,
                          void* stream);

// The folded tcgen05 convolution with its once-per-weights packed filter.
class FoldedConv {
 public:
  enum class Variant { Fold = WF_VARIANT_FOLD, Unfolded = WF_VARIANT_UNFOLDED };
  // Variant::Unfolded runs the same tcgen05 kernel on the unfolded Cin=C input
  // (explicit im2col A tiles) -- the fold-vs-unfolded comparison.
  FoldedConv(const ConvSpec& spec, Dtype in_dtype, std::int64_t factor = 0, std::int64_t group_size = 0,
             Variant variant = Variant::Fold);
  std::size_t packed_bytes() const;
  // Device scratch forward() needs (re-pitched input when W's row pitch is not
  // TMA-addressable, e.g. AlexNet's 227-pixel rows); 0 for zero-copy folds.
  std::size_t workspace_bytes() const { return static_cast<std::size_t>(raw_.workspace_bytes); }
  std::int64_t cout_f() const { return raw_.cout_f; }
  const wf_fold_plan& raw() const { return raw_; }
  const FoldPlan& plan() const { return plan_; }
  const ConvSpec& spec() const { return spec_; }
  Dtype in_dtype() const { return in_; }
  // Expand + pack w (and replicate b when both b and b_rep are given). Once.
  void pack(const void* w, const float* b, void* packed, float* b_rep, void* stream) const;
  // y = ReLU?(conv(x) + b?) ; x in in_dtype, y in out_dtype, NHWC.
  void forward(const void* x, const void* packed, const float* b_rep, void* y, Dtype out_dtype, bool bias, bool relu,
               void* stream, std::uint32_t extra_flags = 0, void* workspace = nullptr) const;
  // The re-pitch pass alone into `workspace` (wf_repitch_input); forward() with
  // WF_EPI_PREPITCHED in extra_flags then skips it.
  void repitch(const void* x, void* workspace, void* stream) const;

 private:
  ConvSpec spec_;
  Dtype in_;
  FoldPlan plan_;
  wf_fold_plan raw_{};
  wf_conv_desc desc_{};
};

}  // namespace widthfold
