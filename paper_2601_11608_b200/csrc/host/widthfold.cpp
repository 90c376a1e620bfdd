// widthfold.cpp -- see widthfold.hpp.
#include "widthfold.hpp"

// fold.hpp spells FoldReason with literal values; they are the C-ABI's.
static_assert(static_cast<int>(widthfold::FoldReason::UnalignedPixel) == WF_REASON_UNALIGNED_PIXEL);
static_assert(static_cast<int>(widthfold::FoldReason::NotProfitable) == WF_REASON_NOT_PROFITABLE);
static_assert(static_cast<int>(widthfold::FoldReason::OutputTail) == WF_REASON_OUTPUT_TAIL);

#include <numeric>
#include <sstream>

namespace widthfold {

void throw_on(wf_status st) {
  if (st == WF_OK) return;
  const std::string msg = wf_last_error();
  switch (st) {
    case WF_SHAPE_MISMATCH: throw ShapeMismatch(msg);
    case WF_DEGENERATE_OUTPUT: throw DegenerateOutput(msg);
    case WF_ILLEGAL_FOLD: throw IllegalFold(msg);
    case WF_NOT_BLOCK_DIAGONAL: throw NotBlockDiagonal(msg);
    case WF_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case WF_UNSUPPORTED: throw Unsupported(msg);
    default: throw CudaError(msg.empty() ? "CUDA error" : msg);
  }
}

void ConvSpec::validate() const {
  if (input_shape.size() != 4) throw ShapeMismatch("conv input must be rank-4 NHWC, got " + shape_str(input_shape));
  if (filter_shape.size() != 4)
    throw ShapeMismatch("conv filter must be rank-4 KHxKWxCinxCout, got " + shape_str(filter_shape));
  for (auto e : input_shape)
    if (e < 1) throw ShapeMismatch("conv input extent < 1: " + shape_str(input_shape));
  for (auto e : filter_shape)
    if (e < 1) throw ShapeMismatch("conv filter extent < 1: " + shape_str(filter_shape));
  if (filter_shape[2] != in_c())
    throw ShapeMismatch("filter Cin " + std::to_string(filter_shape[2]) + " != input Cin " + std::to_string(in_c()));
  if (stride_h < 1 || stride_w < 1) throw ShapeMismatch("strides must be >= 1");
  if (pad_h < 0 || pad_w < 0) throw ShapeMismatch("padding must be >= 0");
  if (in_h() + 2 * pad_h < k_h() || in_w() + 2 * pad_w < k_w() || out_h() < 1 || out_w() < 1)
    throw DegenerateOutput("padding yields empty output for input " + shape_str(input_shape) + ", filter " +
                           shape_str(filter_shape));
}

wf_conv_desc ConvSpec::desc() const {
  return wf_conv_desc{batch(), in_h(), in_w(), in_c(), k_h(), k_w(), out_c(), stride_h, stride_w, pad_h, pad_w};
}

const char* to_string(FoldReason reason) {
  switch (reason) {
    case FoldReason::None: return "None";
    case FoldReason::WidthNotDivisible: return "WidthNotDivisible";
    case FoldReason::KernelSpansFoldAxis: return "KernelSpansFoldAxis";
    case FoldReason::StrideOnFoldAxis: return "StrideOnFoldAxis";
    case FoldReason::AlreadyAligned: return "AlreadyAligned";
    case FoldReason::FactorTooLarge: return "FactorTooLarge";
    case FoldReason::UnsupportedChannels: return "UnsupportedChannels";
    case FoldReason::NotProfitable: return "NotProfitable";
    case FoldReason::UnalignedPixel: return "UnalignedPixel";
    case FoldReason::OutputTail: return "OutputTail";
  }
  return "?";
}

namespace {

FoldPlan fallback_plan(FoldReason r, std::int64_t factor) {
  FoldPlan p;
  p.status = FoldStatus::Fallback;
  p.reason = r;
  p.factor = factor;
  return p;
}

void require_positive(std::int64_t factor, std::int64_t align) {
  if (factor < 1) throw std::invalid_argument("fold factor must be >= 1");
  if (align < 1) throw std::invalid_argument("alignment must be >= 1");
}

}  // namespace

FoldPlan check_legality(const ConvSpec& spec, std::int64_t factor, std::int64_t align) {
  require_positive(factor, align);
  spec.validate();
  // guard order of the reference rule: width, then KW, then stride (src/fold.cpp:51-65)
  if (spec.in_w() % factor != 0) return fallback_plan(FoldReason::WidthNotDivisible, factor);
  if (spec.k_w() != 1) return fallback_plan(FoldReason::KernelSpansFoldAxis, factor);
  if (spec.stride_w != 1) return fallback_plan(FoldReason::StrideOnFoldAxis, factor);
  FoldPlan p;
  p.status = FoldStatus::Apply;
  p.factor = factor;
  p.folded_input_shape = {spec.batch(), spec.in_h(), spec.in_w() / factor, spec.in_c() * factor};
  p.expanded_filter_shape = {spec.k_h(), spec.k_w(), spec.in_c() * factor, factor * spec.out_c()};
  return p;
}

FoldPlan choose_fold_factor(const ConvSpec& spec, std::int64_t align) {
  require_positive(1, align);
  spec.validate();
  if (spec.in_c() % align == 0) return fallback_plan(FoldReason::AlreadyAligned, 1);
  const std::int64_t step = align / std::gcd(spec.in_c(), align);  // smallest aligning factor
  if (step > spec.in_w()) return fallback_plan(FoldReason::FactorTooLarge, step);
  FoldPlan first;
  bool have_first = false;
  for (std::int64_t f = step; f <= spec.in_w(); f += step) {
    FoldPlan p = check_legality(spec, f, align);
    if (p.ok()) return p;
    if (!have_first) {
      first = p;
      have_first = true;
    }
  }
  return first;
}

DevicePlan plan_device_fold(const ConvSpec& spec, std::int64_t factor, std::int64_t group_size, Dtype in_dtype) {
  spec.validate();
  DevicePlan out;
  const wf_conv_desc d = spec.desc();
  throw_on(wf_plan_fold(&d, factor, group_size, static_cast<wf_dtype>(in_dtype), &out.raw));
  out.plan.status = out.raw.status == WF_FOLD_APPLY ? FoldStatus::Apply : FoldStatus::Fallback;
  out.plan.reason = static_cast<FoldReason>(out.raw.reason);
  out.plan.factor = out.raw.f;
  if (out.plan.ok()) {
    const std::int64_t f = out.raw.f;
    out.plan.folded_input_shape = {spec.batch(), spec.in_h(), (spec.in_w() + f - 1) / f, spec.in_c() * f};
    out.plan.expanded_filter_shape = {spec.k_h(), out.raw.kw_f, f * spec.in_c(), out.raw.cout_f};
  }
  return out;
}

MacCount count_macs(const ConvSpec& spec) {
  spec.validate();
  const auto u = [](std::int64_t v) { return static_cast<std::uint64_t>(v); };
  return MacCount{u(spec.batch()) * u(spec.out_h()) * u(spec.out_w()) * u(spec.out_c()) * u(spec.k_h()) *
                  u(spec.k_w()) * u(spec.in_c())};
}

MacReport mac_report(const ConvSpec& spec, const FoldPlan& plan, std::int64_t align) {
  if (!plan.ok()) throw std::invalid_argument("mac_report requires an Apply plan");
  if (align < 1) throw std::invalid_argument("alignment must be >= 1");
  spec.validate();
  MacReport r;
  r.factor = plan.factor;
  r.original = count_macs(spec).macs;
  ConvSpec folded = spec;
  folded.input_shape = plan.folded_input_shape;
  folded.filter_shape = plan.expanded_filter_shape;
  folded.stride_w = 1;
  r.dense_folded = count_macs(folded).macs;
  r.grouped_folded = r.dense_folded / static_cast<std::uint64_t>(plan.factor);
  ConvSpec padded = spec;
  const std::int64_t cin_pad = (spec.in_c() + align - 1) / align * align;
  padded.input_shape[3] = cin_pad;
  padded.filter_shape[2] = cin_pad;
  r.zero_padded = count_macs(padded).macs;
  return r;
}

void conv2d_exact(const float* x, const float* w, float* y, const ConvSpec& spec, void* stream) {
  spec.validate();
  const wf_conv_desc d = spec.desc();
  throw_on(wf_conv_direct_fwd(x, w, y, &d, stream));
}

void conv2d_grouped(const float* x, const float* w_dense, float* y, const ConvSpec& spec, std::int64_t groups,
                    void* stream) {
  spec.validate();
  const wf_conv_desc d = spec.desc();
  throw_on(wf_conv_grouped_fwd(x, w_dense, y, &d, groups, stream));
}

void bias_add(const float* y, const float* b, float* out, std::int64_t n, std::int64_t c, bool relu, void* stream) {
  throw_on(wf_bias_add(y, b, out, n, c, relu ? 1 : 0, stream));
}

void cast_f32(const float* x, void* y, std::int64_t n, Dtype to, void* stream) {
  throw_on(wf_cast_f32(x, y, n, static_cast<wf_dtype>(to), stream));
}

void replicate_bias(const float* b, std::int64_t cout, std::int64_t factor, float* out, void* stream) {
  throw_on(wf_replicate_bias(b, cout, factor, out, stream));
}

Shape folded_filter_shape(const Shape& fs, std::int64_t f, std::int64_t stride_w, std::int64_t pad_w) {
  if (fs.size() != 4) throw IllegalFold("expand_filter wants a rank-4 filter, got " + shape_str(fs));
  if (f < 1) throw std::invalid_argument("fold factor must be >= 1");
  if (stride_w < 1 || f % stride_w != 0) throw IllegalFold("fold factor must be a multiple of stride_w");
  const std::int64_t c0 = -((pad_w + f - 1) / f);
  const std::int64_t num = f - stride_w - pad_w + fs[1] - 1;
  std::int64_t fl = num / f;
  if (num % f != 0 && num < 0) --fl;
  return {fs[0], fl - c0 + 1, f * fs[2], (f / stride_w) * fs[3]};
}

void expand_filter_general(const float* w, const Shape& fs, std::int64_t factor, float* out, void* stream) {
  if (factor < 1) throw std::invalid_argument("fold factor must be >= 1");
  if (fs.size() != 4) throw IllegalFold("expand_filter wants a rank-4 filter, got " + shape_str(fs));
  if (fs[1] != 1)
    throw IllegalFold("cannot expand a filter that spans the fold axis (KW=" + std::to_string(fs[1]) + ")");
  expand_filter_folded(w, fs, factor, 1, 0, out, stream);
}

void expand_filter_folded(const float* w, const Shape& fs, std::int64_t factor, std::int64_t stride_w,
                          std::int64_t pad_w, float* out, void* stream) {
  (void)folded_filter_shape(fs, factor, stride_w, pad_w);  // validates
  const wf_conv_desc d{1, fs[0], fs[1] + factor, fs[2], fs[0], fs[1], fs[3], 1, stride_w, 0, pad_w};
  throw_on(wf_expand_filter_dense(w, &d, factor, out, stream));
}

void check_block_diagonal(const float* w_dense, const Shape& s, std::int64_t groups, void* scratch, void* stream) {
  if (s.size() != 4) throw ShapeMismatch("expanded filter must be rank-4, got " + shape_str(s));
  std::int64_t bad = -1;
  throw_on(wf_check_block_diagonal(w_dense, s[0], s[1], s[2], s[3], groups, scratch, &bad, stream));
}

FoldedConv::FoldedConv(const ConvSpec& spec, Dtype in_dtype, std::int64_t factor, std::int64_t group_size,
                       Variant variant)
    : spec_(spec), in_(in_dtype) {
  DevicePlan dp;
  if (variant == Variant::Unfolded) {
    spec.validate();
    const wf_conv_desc d = spec.desc();
    throw_on(wf_plan_unfolded(&d, static_cast<wf_dtype>(in_dtype), &dp.raw));
    dp.plan.status = dp.raw.status == WF_FOLD_APPLY ? FoldStatus::Apply : FoldStatus::Fallback;
    dp.plan.reason = static_cast<FoldReason>(dp.raw.reason);
    dp.plan.factor = 1;
    if (dp.plan.ok()) {
      dp.plan.folded_input_shape = spec.input_shape;
      dp.plan.expanded_filter_shape = spec.filter_shape;
    }
  } else {
    dp = plan_device_fold(spec, factor, group_size, in_dtype);
  }
  if (!dp.plan.ok())
    throw Unsupported(std::string("width fold not applicable to this conv: ") + to_string(dp.plan.reason) +
                      " (factor " + std::to_string(dp.plan.factor) + ")");
  plan_ = dp.plan;
  raw_ = dp.raw;
  desc_ = spec.desc();
}

std::size_t FoldedConv::packed_bytes() const { return wf_packed_filter_bytes(&raw_); }

void FoldedConv::pack(const void* w, const float* b, void* packed, float* b_rep, void* stream) const {
  throw_on(wf_expand_filter_pack(w, b, &desc_, &raw_, packed, b_rep, stream));
}

void FoldedConv::forward(const void* x, const void* packed, const float* b_rep, void* y, Dtype out_dtype, bool bias,
                         bool relu, void* stream, std::uint32_t extra_flags, void* workspace) const {
  std::uint32_t epi = (bias ? static_cast<std::uint32_t>(WF_EPI_BIAS) : 0u) |
                     (relu ? static_cast<std::uint32_t>(WF_EPI_RELU) : 0u) |
                     (extra_flags & (0xFFFF00u | static_cast<std::uint32_t>(WF_EPI_PREPITCHED)));
  throw_on(wf_conv_fold_fwd_ws(x, workspace, packed, bias ? b_rep : nullptr, y, &desc_, &raw_,
                               static_cast<wf_dtype>(out_dtype), epi, stream));
}

void FoldedConv::repitch(const void* x, void* workspace, void* stream) const {
  throw_on(wf_repitch_input(x, workspace, &desc_, &raw_, stream));
}

}  // namespace widthfold
