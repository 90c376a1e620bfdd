// widthfold.hpp -- C++ host API of widthfold-b200, mirroring the reference
// operator interface (/root/reference/proj/include/widthfold/*.hpp) for the
// folded first-layer conv path, on top of the C-ABI in include/widthfold_b200.h.
//
// Same names, argument meaning and error behaviour as the reference:
//   errors          include/widthfold/errors.hpp:11-30  (exception taxonomy)
//   ConvSpec        include/widthfold/refconv.hpp:14-35 (+ pad_h / pad_w)
//   FoldPlan/Reason include/widthfold/fold.hpp:11-37   (+ UnalignedPixel, OutputTail)
//   check_legality, choose_fold_factor    fold.hpp:42-48 (reference rule, host)
//   count_macs      refconv.hpp:53;  mac_report  blockdiag.hpp:57-67
// Device operations take caller-owned device pointers (no allocation), run on
// a caller-given cudaStream_t and never fall back to the host.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "widthfold_b200.h"

namespace widthfold {

// ---- errors (include/widthfold/errors.hpp:11-30) ------------------------------
struct ShapeMismatch : std::runtime_error { using std::runtime_error::runtime_error; };
struct DegenerateOutput : std::runtime_error { using std::runtime_error::runtime_error; };
struct IllegalFold : std::runtime_error { using std::runtime_error::runtime_error; };
struct NotBlockDiagonal : std::runtime_error { using std::runtime_error::runtime_error; };
// A legal fold the sm_100a kernel cannot execute (no fallback exists).
struct Unsupported : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };

// Turns a wf_status into the matching exception (message from wf_last_error).
void throw_on(wf_status st);

using Shape = std::vector<std::int64_t>;
std::string shape_str(const Shape& s);

enum class Dtype { F32 = WF_F32, TF32 = WF_TF32, BF16 = WF_BF16, F16 = WF_F16 };

// ---- ConvSpec (refconv.hpp:14-35), extended with symmetric padding ------------
struct ConvSpec {
  Shape input_shape;   // (B, H, W, Cin)
  Shape filter_shape;  // (KH, KW, Cin, Cout)
  std::int64_t stride_h = 1;
  std::int64_t stride_w = 1;
  std::int64_t pad_h = 0;
  std::int64_t pad_w = 0;

  std::int64_t batch() const { return input_shape[0]; }
  std::int64_t in_h() const { return input_shape[1]; }
  std::int64_t in_w() const { return input_shape[2]; }
  std::int64_t in_c() const { return input_shape[3]; }
  std::int64_t k_h() const { return filter_shape[0]; }
  std::int64_t k_w() const { return filter_shape[1]; }
  std::int64_t out_c() const { return filter_shape[3]; }
  std::int64_t out_h() const { return (in_h() + 2 * pad_h - k_h()) / stride_h + 1; }
  std::int64_t out_w() const { return (in_w() + 2 * pad_w - k_w()) / stride_w + 1; }
  Shape output_shape() const { return {batch(), out_h(), out_w(), out_c()}; }
  // ShapeMismatch (ranks, Cin, strides, padding) / DegenerateOutput (empty output)
  void validate() const;
  wf_conv_desc desc() const;
};

// ---- fold plan (fold.hpp:11-37) -------------------------------------------------
enum class FoldStatus { Apply, Fallback };
enum class FoldReason {
  None = WF_REASON_NONE,
  WidthNotDivisible = WF_REASON_WIDTH_NOT_DIVISIBLE,
  KernelSpansFoldAxis = WF_REASON_KERNEL_SPANS_FOLD_AXIS,
  StrideOnFoldAxis = WF_REASON_STRIDE_ON_FOLD_AXIS,
  AlreadyAligned = WF_REASON_ALREADY_ALIGNED,
  FactorTooLarge = WF_REASON_FACTOR_TOO_LARGE,
  UnsupportedChannels = WF_REASON_UNSUPPORTED_CHANNELS,
  NotProfitable = WF_REASON_NOT_PROFITABLE,
  UnalignedPixel = WF_REASON_UNALIGNED_PIXEL,
  OutputTail = WF_REASON_OUTPUT_TAIL,
};
const char* to_string(FoldReason reason);

struct FoldPlan {
  FoldStatus status = FoldStatus::Fallback;
  FoldReason reason = FoldReason::None;
  std::int64_t factor = 1;
  int axis = 2;                 // W in NHWC
  Shape folded_input_shape;     // (B, H, W/F, Cin*F) when Apply
  Shape expanded_filter_shape;  // reference rule: (KH, KW, Cin*F, F*Cout); generalized: (KH, KW', F*Cin, r*Cout)
  bool ok() const { return status == FoldStatus::Apply; }
};

// Reference legality (src/fold.cpp:51-90): Apply iff W%F==0, KW==1, stride_w==1.
// std::invalid_argument for F < 1 or align < 1. Failures are values.
FoldPlan check_legality(const ConvSpec& spec, std::int64_t factor, std::int64_t align);
FoldPlan choose_fold_factor(const ConvSpec& spec, std::int64_t align);

// Generalized device fold: KW > 1, stride, padding.
// factor == 0 picks the factor; returns the raw device schedule too.
struct DevicePlan {
  FoldPlan plan;
  wf_fold_plan raw{};
};
DevicePlan plan_device_fold(const ConvSpec& spec, std::int64_t factor, std::int64_t group_size, Dtype in_dtype);

// ---- MAC accounting (refconv.cpp:116-122, blockdiag.cpp:189-217) -------------------
std::uint64_t count_macs(const ConvSpec& spec);
struct MacReport {
  std::uint64_t original = 0;
  std::uint64_t dense_folded = 0;
  std::uint64_t grouped_folded = 0;
  std::uint64_t zero_padded = 0;
  std::int64_t factor = 1;
};
// Reference rule: requires plan.ok() (std::invalid_argument otherwise).
MacReport mac_report(const ConvSpec& spec, const FoldPlan& plan, std::int64_t align);

// ---- device operations ------------------------------------------------------------
// Exact-order fp32 conv2d + optional bias/ReLU (reference conv2d/bias_add bits).
void conv2d_exact(const float* x, const float* w, float* y, const ConvSpec& spec, void* stream);
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

 private:
  ConvSpec spec_;
  Dtype in_;
  FoldPlan plan_;
  wf_fold_plan raw_{};
  wf_conv_desc desc_{};
};

}  // namespace widthfold
