// widthfold/fold.hpp -- the width-fold rewrite, same include path and
// signatures as the reference (/root/reference/proj/include/widthfold/fold.hpp:11-96).
//
// The index transforms (fold_input[_general], unfold_input_general,
// reconstruct_output) are the row-major identity -- on the device they are
// zero-copy views; on a DenseTensor value they are reshapes. The filter
// expansion and the bias replication run as device kernels
// (wf_expand_filter_dense, wf_replicate_bias) and come back bit-exact.
// check_legality / choose_fold_factor keep the reference rule (W % F == 0,
// KW == 1, stride_w == 1); the generalized device fold (KW > 1, stride,
// padding) is widthfold::plan_device_fold in the device API (widthfold.hpp).
#pragma once

#include <cstdint>
#include <string>

#include "widthfold/refconv.hpp"
#include "widthfold/tensor.hpp"

namespace widthfold {

enum class FoldStatus { Apply, Fallback };

enum class FoldReason {
  None = 0,
  WidthNotDivisible = 1,
  KernelSpansFoldAxis = 2,
  StrideOnFoldAxis = 3,
  AlreadyAligned = 4,
  FactorTooLarge = 5,
  UnsupportedChannels = 6,
  NotProfitable = 7,
  UnalignedPixel = 8,  // device fold: f*C*elem not a multiple of the MMA K-step
  OutputTail = 9,      // reserved
};

const char* to_string(FoldReason reason);

struct FoldPlan {
  FoldStatus status = FoldStatus::Fallback;
  FoldReason reason = FoldReason::None;
  std::int64_t factor = 1;
  int axis = 2;                 // W in NHWC
  Shape folded_input_shape;     // (B, H, W/F, Cin*F) when Apply
  Shape expanded_filter_shape;  // reference rule (KH, KW, Cin*F, F*Cout); device fold (KH, KW', F*Cin, r*Cout)

  bool ok() const { return status == FoldStatus::Apply; }
};

// Legality is a value, never an error (std::invalid_argument for F < 1 / align < 1).
FoldPlan check_legality(const ConvSpec& spec, std::int64_t factor, std::int64_t align);
FoldPlan choose_fold_factor(const ConvSpec& spec, std::int64_t align);

DenseTensor fold_input(const DenseTensor& x, std::int64_t factor);
DenseTensor fold_input_general(const DenseTensor& x, std::int64_t factor);
DenseTensor unfold_input_general(const DenseTensor& x_f, std::int64_t factor);
DenseTensor expand_filter(const DenseTensor& w, std::int64_t factor);
DenseTensor expand_filter_general(const DenseTensor& w, std::int64_t factor);
DenseTensor replicate_bias(const DenseTensor& b, std::int64_t factor);
DenseTensor reconstruct_output(const DenseTensor& y_folded, std::int64_t factor);

struct FoldResult {
  FoldPlan plan;
  DenseTensor input;   // folded on Apply, original on Fallback
  DenseTensor filter;  // expanded on Apply, original on Fallback
  DenseTensor bias;    // replicated on Apply, original on Fallback
};

// Total: legality failures return Fallback plus the untouched inputs.
FoldResult apply_width_fold(const DenseTensor& x, const DenseTensor& w, const DenseTensor& b, std::int64_t factor);
FoldResult apply_width_fold_general(const DenseTensor& x, const DenseTensor& w, const DenseTensor& b,
                                    std::int64_t factor);

}  // namespace widthfold
