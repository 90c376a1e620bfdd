// dense_api.cpp -- the reference's DenseTensor-valued operator API
// (include/widthfold/{tensor,refconv,fold,blockdiag}.hpp), each operation
// running on the B200 through the C-ABI.
//
// Reference semantics followed (file:line under /root/reference/proj):
//   DenseTensor, reshape, max_abs_diff          src/tensor.cpp:9-120
//   conv2d / bias_add / conv1d_h                src/refconv.cpp:34-114
//   fold_input[_general], unfold_input_general,
//   expand_filter[_general], replicate_bias,
//   reconstruct_output, apply_width_fold[_general]  src/fold.cpp:92-317
//   BlockDiagFilter, grouped_conv               src/blockdiag.cpp:8-187
// Same guard order, exception types and messages. Values cross the boundary
// as host DenseTensors; the arithmetic (the exact-order fp32 conv, bias_add,
// the filter expansion, bias replication and the strict-zero block check)
// runs in the device kernels behind wf_* -- there is no host compute path.
// The index transforms of the fold are the row-major identity (zero-copy
// views on the device), so on a value they are reshapes.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <sstream>

#include "widthfold.hpp"

namespace widthfold {

// ---------------------------------------------------------------- tensor.hpp
std::int64_t numel(const Shape& shape) {
  std::int64_t n = 1;
  for (auto e : shape) n *= e;
  return n;
}

std::string shape_str(const Shape& shape) {
  std::ostringstream os;
  os << '(';
  for (std::size_t i = 0; i < shape.size(); ++i) os << (i ? "," : "") << shape[i];
  os << ')';
  return os.str();
}

Shape strides_of(const Shape& shape) {
  Shape st(shape.size(), 1);
  for (std::size_t i = shape.size(); i-- > 1;) st[i - 1] = st[i] * shape[i];
  return st;
}

DenseTensor::DenseTensor(Shape shape, std::vector<float> data) : shape_(std::move(shape)), data_(std::move(data)) {
  for (auto e : shape_)
    if (e < 1) throw ShapeMismatch("tensor extent must be >= 1, got shape " + shape_str(shape_));
  if (numel(shape_) != static_cast<std::int64_t>(data_.size()))
    throw ShapeMismatch("shape " + shape_str(shape_) + " wants " + std::to_string(numel(shape_)) +
                        " elements, got " + std::to_string(data_.size()));
}

DenseTensor DenseTensor::zeros(Shape shape) { return full(std::move(shape), 0.0f); }

DenseTensor DenseTensor::full(Shape shape, float value) {
  const auto n = numel(shape);
  return DenseTensor(std::move(shape), std::vector<float>(static_cast<std::size_t>(n < 0 ? 0 : n), value));
}

std::int64_t DenseTensor::offset(std::span<const std::int64_t> coord) const {
  if (coord.size() != shape_.size())
    throw ShapeMismatch("coordinate rank " + std::to_string(coord.size()) + " does not match tensor rank " +
                        std::to_string(shape_.size()));
  std::int64_t off = 0;
  for (std::size_t i = 0; i < coord.size(); ++i) {
    if (coord[i] < 0 || coord[i] >= shape_[i])
      throw ShapeMismatch("coordinate out of range for shape " + shape_str(shape_));
    off = off * shape_[i] + coord[i];
  }
  return off;
}

float DenseTensor::at(std::span<const std::int64_t> coord) const {
  return data_[static_cast<std::size_t>(offset(coord))];
}

float DenseTensor::at(std::initializer_list<std::int64_t> coord) const {
  return at(std::span<const std::int64_t>(coord.begin(), coord.size()));
}

bool DenseTensor::bitwise_equal(const DenseTensor& other) const {
  return shape_ == other.shape_ && data_.size() == other.data_.size() &&
         (data_.empty() || std::memcmp(data_.data(), other.data_.data(), data_.size() * sizeof(float)) == 0);
}

DenseTensor reshape(const DenseTensor& t, Shape new_shape) {
  if (numel(new_shape) != t.size())
    throw ShapeMismatch("cannot reshape " + shape_str(t.shape()) + " to " + shape_str(new_shape) +
                        ": element counts differ");
  return DenseTensor(std::move(new_shape), std::vector<float>(t.data().begin(), t.data().end()));
}

float max_abs_diff(const DenseTensor& a, const DenseTensor& b) {
  if (a.shape() != b.shape())
    throw ShapeMismatch("max_abs_diff shapes differ: " + shape_str(a.shape()) + " vs " + shape_str(b.shape()));
  float worst = 0.0f;
  const auto da = a.data(), db = b.data();
  for (std::size_t i = 0; i < da.size(); ++i) {
    const float d = std::fabs(da[i] - db[i]);
    if (std::isnan(d)) return d;
    worst = d > worst ? d : worst;
  }
  return worst;
}

// ---------------------------------------------------------------- device staging
namespace {

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// One device allocation; operations use the legacy default stream, so the
// synchronous copies order them.
class DeviceBuffer {
 public:
  explicit DeviceBuffer(std::size_t bytes) {
    if (bytes) cuda_ok(cudaMalloc(&p_, bytes), "cudaMalloc");
  }
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_) { o.p_ = nullptr; }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  ~DeviceBuffer() {
    if (p_) cudaFree(p_);
  }
  float* f() const { return static_cast<float*>(p_); }
  void* get() const { return p_; }

 private:
  void* p_ = nullptr;
};

std::size_t bytes_of(std::int64_t n) { return static_cast<std::size_t>(n) * sizeof(float); }

DeviceBuffer to_device(const DenseTensor& t) {
  DeviceBuffer d(bytes_of(t.size()));
  if (t.size()) cuda_ok(cudaMemcpy(d.get(), t.data().data(), bytes_of(t.size()), cudaMemcpyHostToDevice), "H2D");
  return d;
}

DenseTensor to_host(const DeviceBuffer& d, Shape shape) {
  std::vector<float> out(static_cast<std::size_t>(numel(shape)));
  if (!out.empty())
    cuda_ok(cudaMemcpy(out.data(), d.get(), bytes_of(static_cast<std::int64_t>(out.size())), cudaMemcpyDeviceToHost),
            "D2H");
  return DenseTensor(std::move(shape), std::move(out));
}

void require_factor(std::int64_t factor) {
  if (factor < 1) throw std::invalid_argument("fold factor must be >= 1");
}

}  // namespace

// ---------------------------------------------------------------- refconv.hpp
DenseTensor conv2d(const DenseTensor& x, const DenseTensor& w, const ConvSpec& spec) {
  spec.validate();
  if (x.shape() != spec.input_shape)
    throw ShapeMismatch("conv input " + shape_str(x.shape()) + " does not match spec " +
                        shape_str(spec.input_shape));
  if (w.shape() != spec.filter_shape)
    throw ShapeMismatch("conv filter " + shape_str(w.shape()) + " does not match spec " +
                        shape_str(spec.filter_shape));
  const DeviceBuffer xd = to_device(x), wd = to_device(w);
  const Shape os = spec.output_shape();
  DeviceBuffer yd(bytes_of(numel(os)));
  conv2d_exact(xd.f(), wd.f(), yd.f(), spec, nullptr);
  return to_host(yd, os);
}

DenseTensor bias_add(const DenseTensor& y, const DenseTensor& b) {
  if (y.rank() < 1 || b.rank() != 1 || b.shape()[0] != y.shape().back())
    throw ShapeMismatch("bias length " + shape_str(b.shape()) + " does not match channel extent of " +
                        shape_str(y.shape()));
  const DeviceBuffer yd = to_device(y), bd = to_device(b);
  DeviceBuffer od(bytes_of(y.size()));
  bias_add(yd.f(), bd.f(), od.f(), y.size(), b.shape()[0], false, nullptr);
  return to_host(od, y.shape());
}

DenseTensor conv1d_h(const DenseTensor& x, const DenseTensor& w, float bias) {
  if (x.rank() != 3 || x.shape()[2] != 1)
    throw ShapeMismatch("conv1d_h input must be (H, W, 1), got " + shape_str(x.shape()));
  if (w.rank() != 1) throw ShapeMismatch("conv1d_h kernel must be rank-1, got " + shape_str(w.shape()));
  const std::int64_t H = x.shape()[0], W = x.shape()[1], K = w.shape()[0];
  if (K > H) throw ShapeMismatch("kernel length exceeds height");
  const ConvSpec spec{{1, H, W, 1}, {K, 1, 1, 1}, 1, 1};
  const DenseTensor y = bias_add(conv2d(reshape(x, {1, H, W, 1}), reshape(w, {K, 1, 1, 1}), spec),
                                 DenseTensor({1}, {bias}));
  return reshape(y, {spec.out_h(), W, 1});
}

// ---------------------------------------------------------------- fold.hpp
DenseTensor fold_input(const DenseTensor& x, std::int64_t factor) {
  require_factor(factor);
  if (x.rank() != 4) throw IllegalFold("fold_input wants a rank-4 NHWC tensor, got " + shape_str(x.shape()));
  const Shape& s = x.shape();
  if (s[3] != 1) throw IllegalFold("fold_input requires Cin == 1, got " + std::to_string(s[3]));
  if (s[2] % factor != 0)
    throw IllegalFold("width " + std::to_string(s[2]) + " not divisible by " + std::to_string(factor));
  return reshape(x, {s[0], s[1], s[2] / factor, factor});
}

DenseTensor fold_input_general(const DenseTensor& x, std::int64_t factor) {
  require_factor(factor);
  if (x.rank() != 4)
    throw IllegalFold("fold_input_general wants a rank-4 NHWC tensor, got " + shape_str(x.shape()));
  const Shape& s = x.shape();
  if (s[2] % factor != 0)
    throw IllegalFold("width " + std::to_string(s[2]) + " not divisible by " + std::to_string(factor));
  return reshape(x, {s[0], s[1], s[2] / factor, s[3] * factor});  // X_f[b,h,w',f*C+c] = X[b,h,F*w'+f,c]
}

DenseTensor unfold_input_general(const DenseTensor& x_f, std::int64_t factor) {
  require_factor(factor);
  if (x_f.rank() != 4)
    throw IllegalFold("unfold_input_general wants a rank-4 tensor, got " + shape_str(x_f.shape()));
  const Shape& s = x_f.shape();
  if (s[3] % factor != 0)
    throw IllegalFold("channel extent " + std::to_string(s[3]) + " not divisible by " + std::to_string(factor));
  return reshape(x_f, {s[0], s[1], s[2] * factor, s[3] / factor});
}

DenseTensor expand_filter(const DenseTensor& w, std::int64_t factor) {
  if (w.rank() != 4 || w.shape()[2] != 1)
    throw IllegalFold("expand_filter wants a (KH, 1, 1, Cout) filter, got " + shape_str(w.shape()));
  return expand_filter_general(w, factor);
}

DenseTensor expand_filter_general(const DenseTensor& w, std::int64_t factor) {
  require_factor(factor);
  if (w.rank() != 4) throw IllegalFold("expand_filter wants a rank-4 filter, got " + shape_str(w.shape()));
  const Shape& s = w.shape();
  if (s[1] != 1)
    throw IllegalFold("cannot expand a filter that spans the fold axis (KW=" + std::to_string(s[1]) + ")");
  const DeviceBuffer wd = to_device(w);
  const Shape os{s[0], 1, s[2] * factor, s[3] * factor};
  DeviceBuffer od(bytes_of(numel(os)));
  expand_filter_general(wd.f(), s, factor, od.f(), nullptr);
  return to_host(od, os);
}

DenseTensor replicate_bias(const DenseTensor& b, std::int64_t factor) {
  require_factor(factor);
  if (b.rank() != 1) throw ShapeMismatch("bias must be rank-1, got " + shape_str(b.shape()));
  const DeviceBuffer bd = to_device(b);
  DeviceBuffer od(bytes_of(b.size() * factor));
  replicate_bias(bd.f(), b.shape()[0], factor, od.f(), nullptr);
  return to_host(od, {b.shape()[0] * factor});
}

DenseTensor reconstruct_output(const DenseTensor& y_folded, std::int64_t factor) {
  require_factor(factor);
  if (y_folded.rank() != 4)
    throw ShapeMismatch("reconstruct_output wants a rank-4 tensor, got " + shape_str(y_folded.shape()));
  const Shape& s = y_folded.shape();
  if (s[3] % factor != 0)
    throw ShapeMismatch("channel extent " + std::to_string(s[3]) + " not divisible by fold factor " +
                        std::to_string(factor));
  return reshape(y_folded, {s[0], s[1], s[2] * factor, s[3] / factor});
}

namespace {

// src/fold.cpp:263-304: shape guards throw, legality failures fall back.
FoldResult fold_with_guard(const DenseTensor& x, const DenseTensor& w, const DenseTensor& b, std::int64_t factor,
                           bool single_channel) {
  require_factor(factor);
  if (x.rank() != 4) throw ShapeMismatch("apply_width_fold input must be rank-4 NHWC, got " + shape_str(x.shape()));
  if (w.rank() != 4) throw ShapeMismatch("apply_width_fold filter must be rank-4, got " + shape_str(w.shape()));
  if (b.rank() != 1 || b.shape()[0] != w.shape()[3])
    throw ShapeMismatch("bias " + shape_str(b.shape()) + " does not match filter Cout " +
                        std::to_string(w.shape()[3]));
  if (x.shape()[3] != w.shape()[2])
    throw ShapeMismatch("input Cin " + std::to_string(x.shape()[3]) + " != filter Cin " +
                        std::to_string(w.shape()[2]));
  auto fall = [&](FoldReason reason) {
    FoldResult r{FoldPlan{}, x, w, b};
    r.plan.reason = reason;
    r.plan.factor = factor;
    return r;
  };
  if (x.shape()[2] % factor != 0) return fall(FoldReason::WidthNotDivisible);
  if (single_channel && x.shape()[3] != 1) return fall(FoldReason::UnsupportedChannels);
  if (w.shape()[1] != 1) return fall(FoldReason::KernelSpansFoldAxis);
  FoldResult r;
  r.plan.status = FoldStatus::Apply;
  r.plan.factor = factor;
  r.plan.folded_input_shape = {x.shape()[0], x.shape()[1], x.shape()[2] / factor, x.shape()[3] * factor};
  r.plan.expanded_filter_shape = {w.shape()[0], w.shape()[1], w.shape()[2] * factor, factor * w.shape()[3]};
  r.input = single_channel ? fold_input(x, factor) : fold_input_general(x, factor);
  r.filter = expand_filter_general(w, factor);
  r.bias = replicate_bias(b, factor);
  return r;
}

}  // namespace

FoldResult apply_width_fold(const DenseTensor& x, const DenseTensor& w, const DenseTensor& b, std::int64_t factor) {
  return fold_with_guard(x, w, b, factor, true);
}

FoldResult apply_width_fold_general(const DenseTensor& x, const DenseTensor& w, const DenseTensor& b,
                                    std::int64_t factor) {
  return fold_with_guard(x, w, b, factor, false);
}

// ---------------------------------------------------------------- blockdiag.hpp
BlockDiagFilter::BlockDiagFilter(std::vector<DenseTensor> blocks, std::int64_t num_blocks)
    : blocks_(std::move(blocks)), num_blocks_(num_blocks) {
  if (blocks_.empty() || num_blocks_ < 1) throw ShapeMismatch("BlockDiagFilter needs at least one block");
  for (const auto& b : blocks_) {
    if (b.rank() != 4) throw ShapeMismatch("block must be rank-4 KHxKWxCinxCout, got " + shape_str(b.shape()));
    if (b.shape() != blocks_.front().shape()) throw ShapeMismatch("all blocks must share one shape");
  }
}

BlockDiagFilter BlockDiagFilter::from_expanded(const DenseTensor& dense, std::int64_t num_blocks) {
  if (dense.rank() != 4) throw ShapeMismatch("expanded filter must be rank-4, got " + shape_str(dense.shape()));
  const Shape& s = dense.shape();
  const std::int64_t KH = s[0], KW = s[1], Cif = s[2], Cof = s[3];
  if (num_blocks < 1 || Cif % num_blocks != 0 || Cof % num_blocks != 0)
    throw ShapeMismatch("channel extents " + std::to_string(Cif) + "x" + std::to_string(Cof) +
                        " not divisible into " + std::to_string(num_blocks) + " blocks");
  {  // strict-zero check on the device (first offending entry in flat order)
    const DeviceBuffer dd = to_device(dense);
    DeviceBuffer scratch(8);
    std::int64_t bad = -1;
    const wf_status st = wf_check_block_diagonal(dd.f(), KH, KW, Cif, Cof, num_blocks, scratch.get(), &bad, nullptr);
    if (st == WF_NOT_BLOCK_DIAGONAL && bad >= 0) {
      const std::int64_t co = bad % Cof, ci = bad / Cof % Cif, kw = bad / (Cof * Cif) % KW, kh = bad / (Cof * Cif * KW);
      throw NotBlockDiagonal("off-diagonal entry at (kh=" + std::to_string(kh) + ", kw=" + std::to_string(kw) +
                             ", cin=" + std::to_string(ci) + ", cout=" + std::to_string(co) + ") is nonzero");
    }
    throw_on(st);
  }
  const std::int64_t Cib = Cif / num_blocks, Cob = Cof / num_blocks;
  const float* d = dense.data().data();
  std::vector<DenseTensor> blocks;
  for (std::int64_t g = 0; g < num_blocks; ++g) {
    std::vector<float> blk(static_cast<std::size_t>(KH * KW * Cib * Cob));
    std::size_t o = 0;
    for (std::int64_t r = 0; r < KH * KW; ++r)
      for (std::int64_t c = 0; c < Cib; ++c)
        for (std::int64_t co = 0; co < Cob; ++co) blk[o++] = d[(r * Cif + g * Cib + c) * Cof + g * Cob + co];
    blocks.emplace_back(Shape{KH, KW, Cib, Cob}, std::move(blk));
  }
  bool same = true;
  for (std::size_t g = 1; g < blocks.size() && same; ++g) same = blocks[g].bitwise_equal(blocks[0]);
  if (same && num_blocks > 1) return shared(std::move(blocks[0]), num_blocks);
  return BlockDiagFilter(std::move(blocks), num_blocks);
}

BlockDiagFilter BlockDiagFilter::shared(DenseTensor block, std::int64_t num_blocks) {
  std::vector<DenseTensor> blocks;
  blocks.push_back(std::move(block));
  return BlockDiagFilter(std::move(blocks), num_blocks);
}

BlockDiagFilter BlockDiagFilter::from_blocks(std::vector<DenseTensor> blocks) {
  const auto n = static_cast<std::int64_t>(blocks.size());
  return BlockDiagFilter(std::move(blocks), n);
}

const DenseTensor& BlockDiagFilter::block(std::int64_t i) const {
  if (i < 0 || i >= num_blocks_) throw ShapeMismatch("block index out of range");
  return blocks_.size() == 1 ? blocks_[0] : blocks_[static_cast<std::size_t>(i)];
}

Shape BlockDiagFilter::logical_shape() const {
  const Shape& b = blocks_.front().shape();
  return {b[0], b[1], b[2] * num_blocks_, b[3] * num_blocks_};
}

std::int64_t BlockDiagFilter::stored_floats() const { return num_blocks_ * blocks_.front().size(); }

DenseTensor BlockDiagFilter::densify() const {
  const Shape ls = logical_shape();
  const std::int64_t KHW = ls[0] * ls[1], Cif = ls[2], Cof = ls[3];
  const std::int64_t Cib = Cif / num_blocks_, Cob = Cof / num_blocks_;
  std::vector<float> out(static_cast<std::size_t>(numel(ls)), 0.0f);
  for (std::int64_t g = 0; g < num_blocks_; ++g) {
    const float* src = block(g).data().data();
    for (std::int64_t r = 0; r < KHW; ++r)
      for (std::int64_t c = 0; c < Cib; ++c)
        for (std::int64_t co = 0; co < Cob; ++co)
          out[(r * Cif + g * Cib + c) * Cof + g * Cob + co] = src[(r * Cib + c) * Cob + co];
  }
  return DenseTensor(ls, std::move(out));
}

// The grouped conv skips the off-block terms and keeps the surviving order
// (src/blockdiag.cpp:138-187): on the device, the exact-order conv kernel in
// grouped mode over the densified filter (diagonal blocks only are read).
DenseTensor grouped_conv(const DenseTensor& x_f, const BlockDiagFilter& bd, const ConvSpec& spec) {
  spec.validate();
  const Shape ls = bd.logical_shape();
  if (x_f.shape() != spec.input_shape || ls != spec.filter_shape)
    throw ShapeMismatch("grouped_conv shapes do not match spec: input " + shape_str(x_f.shape()) + ", filter " +
                        shape_str(ls) + ", spec " + shape_str(spec.input_shape) + "/" +
                        shape_str(spec.filter_shape));
  const DenseTensor dense = bd.densify();
  const DeviceBuffer xd = to_device(x_f), wd = to_device(dense);
  const Shape os = spec.output_shape();
  DeviceBuffer yd(bytes_of(numel(os)));
  conv2d_grouped(xd.f(), wd.f(), yd.f(), spec, bd.num_blocks(), nullptr);
  return to_host(yd, os);
}

}  // namespace widthfold
