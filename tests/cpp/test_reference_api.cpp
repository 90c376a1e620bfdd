// test_reference_api.cpp -- a reference C++ caller, compiled unchanged against
// widthfold-b200's headers at the reference's include paths
// (#include "widthfold/...") and linked with ../../paper_2601_11608_b200/libwidthfold.so.
//
// The calls below are the reference's own call-site shapes: the acceptance
// pipelines (tests/acceptance/acceptance_main.cpp:46-55), the golden single
// conv and the oracle-equivalence sweep (:60-124), the expand_filter /
// replicate_bias / fold unit cases (tests/unit/test_fold.cpp:152-240), the
// BlockDiagFilter and grouped_conv contract (include/widthfold/blockdiag.hpp)
// and the MAC report (acceptance_main.cpp:472-509). Every operation runs on
// the B200 behind the C-ABI.
//
//   test_reference_api [--host-only] [golden_dir]
// --host-only runs just the checks that need no GPU (values, errors,
// legality, MAC accounting). golden_dir holds <key>.f32 + <key>.shape files
// dumped from tests/golden/appendix_a.npz (tests/test_cpp_api.py), the
// Appendix-A vectors the reference's own pybind module produced.
// Prints one [PASS]/[FAIL] line per criterion; exit code = failures.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <functional>
#include <iostream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "widthfold/blockdiag.hpp"
#include "widthfold/fold.hpp"
#include "widthfold/refconv.hpp"
#include "widthfold/tensor.hpp"

using namespace widthfold;

namespace {

struct Failure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void require(bool ok, const std::string& what) {
  if (!ok) throw Failure(what);
}

template <class E, class F>
void require_throws(F&& f, const std::string& what) {
  try {
    f();
  } catch (const E&) {
    return;
  } catch (const std::exception& e) {
    throw Failure(what + " (threw the wrong type: " + e.what() + ")");
  }
  throw Failure(what + " (did not throw)");
}

// Seeded data: the reference test generator's value maps (small integers in
// [-4, 4], uniform floats in [-1, 1)) over std::mt19937.
struct Rng {
  std::mt19937 rng;
  explicit Rng(std::uint32_t seed) : rng(seed) {}
  DenseTensor ints(const Shape& s) {
    std::vector<float> v(static_cast<std::size_t>(numel(s)));
    for (auto& e : v) e = static_cast<float>(static_cast<int>(rng() % 9) - 4);
    return DenseTensor(s, std::move(v));
  }
  DenseTensor floats(const Shape& s) {
    std::vector<float> v(static_cast<std::size_t>(numel(s)));
    for (auto& e : v) e = static_cast<float>(rng() >> 8) * (2.0f / 16777216.0f) - 1.0f;
    return DenseTensor(s, std::move(v));
  }
};

// Independent host oracle: six nested loops, kh -> kw -> ci, fresh index math.
DenseTensor naive_conv_bias(const DenseTensor& x, const DenseTensor& w, const DenseTensor& b) {
  const Shape& xs = x.shape();
  const Shape& ws = w.shape();
  const std::int64_t OH = xs[1] - ws[0] + 1, OW = xs[2] - ws[1] + 1;
  std::vector<float> out;
  for (std::int64_t n = 0; n < xs[0]; ++n)
    for (std::int64_t oh = 0; oh < OH; ++oh)
      for (std::int64_t ow = 0; ow < OW; ++ow)
        for (std::int64_t oc = 0; oc < ws[3]; ++oc) {
          float acc = 0.0f;
          for (std::int64_t kh = 0; kh < ws[0]; ++kh)
            for (std::int64_t kw = 0; kw < ws[1]; ++kw)
              for (std::int64_t ci = 0; ci < ws[2]; ++ci)
                acc += x.at({n, oh + kh, ow + kw, ci}) * w.at({kh, kw, ci, oc});
          out.push_back(acc + b.at({oc}));
        }
  return DenseTensor({xs[0], OH, OW, ws[3]}, std::move(out));
}

// acceptance_main.cpp:46-55
DenseTensor pipeline_original(const DenseTensor& x, const DenseTensor& w, const DenseTensor& b) {
  return bias_add(conv2d(x, w, ConvSpec{x.shape(), w.shape()}), b);
}

DenseTensor pipeline_folded(const FoldResult& r) {
  const ConvSpec spec{r.input.shape(), r.filter.shape()};
  return reconstruct_output(bias_add(conv2d(r.input, r.filter, spec), r.bias), r.plan.factor);
}

std::string g_golden;

DenseTensor load_golden(const std::string& key) {
  std::ifstream sf(g_golden + "/" + key + ".shape");
  require(bool(sf), "missing golden " + key);
  Shape s;
  for (std::int64_t e; sf >> e;) s.push_back(e);
  std::vector<float> v(static_cast<std::size_t>(numel(s)));
  std::ifstream df(g_golden + "/" + key + ".f32", std::ios::binary);
  df.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(float)));
  require(bool(df), "short golden blob " + key);
  return DenseTensor(s, std::move(v));
}

// ---------------------------------------------------------------- host-only criteria
std::string values_and_errors() {
  const DenseTensor t({2, 3}, {1, 2, 3, 4, 5, -0.0f});
  require(t.at({1, 2}) == 0.0f && std::signbit(t.at({1, 2})), "at() keeps -0.0");
  require(!t.bitwise_equal(DenseTensor({2, 3}, {1, 2, 3, 4, 5, 0.0f})), "bitwise_equal distinguishes -0.0");
  require(reshape(t, {3, 2}).bitwise_equal(DenseTensor({3, 2}, {1, 2, 3, 4, 5, -0.0f})), "reshape keeps data");
  require(strides_of({2, 3, 4}) == Shape{12, 4, 1}, "row-major strides");
  require(shape_str({1, 32, 64, 1}) == "(1,32,64,1)", "shape_str format");
  require(std::isnan(max_abs_diff(t, DenseTensor({2, 3}, {1, 2, 3, 4, NAN, 0}))), "NaN propagates");
  require(max_abs_diff(t, DenseTensor::full({2, 3}, 1.0f)) == 4.0f, "max_abs_diff");
  require_throws<ShapeMismatch>([] { DenseTensor({2, 2}, {1, 2, 3}); }, "count mismatch");
  require_throws<ShapeMismatch>([] { DenseTensor({0, 2}, {}); }, "zero extent");
  require_throws<ShapeMismatch>([&] { (void)t.at({2, 0}); }, "out-of-range coordinate");
  require_throws<ShapeMismatch>([&] { (void)reshape(t, {4, 2}); }, "reshape count");
  require_throws<ShapeMismatch>([] { ConvSpec{{1, 8, 8}, {3, 1, 1, 1}}.validate(); }, "rank-3 input");
  require_throws<DegenerateOutput>([] { ConvSpec{{1, 2, 8, 1}, {3, 1, 1, 1}}.validate(); }, "empty output");
  require_throws<ShapeMismatch>([] { ConvSpec{{1, 8, 8, 2}, {3, 1, 1, 1}}.validate(); }, "Cin mismatch");
  require_throws<std::invalid_argument>([] { check_legality(ConvSpec{{1, 8, 8, 1}, {3, 1, 1, 1}}, 0, 8); },
                                        "factor 0");
  require_throws<IllegalFold>([] { fold_input(DenseTensor::zeros({1, 2, 7, 1}), 2); }, "fold_input W % F");
  require_throws<IllegalFold>([] { fold_input(DenseTensor::zeros({1, 2, 8, 2}), 2); }, "fold_input Cin != 1");
  require_throws<ShapeMismatch>([] { reconstruct_output(DenseTensor::zeros({1, 2, 3, 5}), 2); },
                                "reconstruct_output Cout % F");
  require_throws<ShapeMismatch>(
      [] { apply_width_fold(DenseTensor::zeros({1, 4, 8, 1}), DenseTensor::zeros({3, 1, 1, 2}),
                            DenseTensor::zeros({3}), 2); },
      "apply_width_fold bias length");
  return "DenseTensor value semantics and the error taxonomy";
}

std::string legality_and_macs() {
  const ConvSpec spec{{1, 32, 64, 1}, {5, 1, 1, 1}, 1, 1};
  const FoldPlan p = check_legality(spec, 8, 8);
  require(p.ok() && p.folded_input_shape == Shape({1, 32, 8, 8}) && p.expanded_filter_shape == Shape({5, 1, 8, 8}),
          "Appendix-A legality");
  require(check_legality(ConvSpec{{1, 4, 7, 1}, {3, 1, 1, 1}}, 8, 8).reason == FoldReason::WidthNotDivisible,
          "WidthNotDivisible");
  require(check_legality(ConvSpec{{1, 8, 8, 1}, {3, 3, 1, 1}}, 2, 8).reason == FoldReason::KernelSpansFoldAxis,
          "KernelSpansFoldAxis");
  require(check_legality(ConvSpec{{1, 8, 8, 1}, {3, 1, 1, 1}, 1, 2}, 2, 8).reason == FoldReason::StrideOnFoldAxis,
          "StrideOnFoldAxis");
  require(choose_fold_factor(ConvSpec{{1, 8, 8, 8}, {3, 1, 8, 1}}, 8).reason == FoldReason::AlreadyAligned,
          "AlreadyAligned");
  require(choose_fold_factor(ConvSpec{{1, 8, 4, 1}, {3, 1, 1, 1}}, 8).reason == FoldReason::FactorTooLarge,
          "FactorTooLarge");
  require(std::string(to_string(FoldReason::NotProfitable)) == "NotProfitable", "to_string");
  require(count_macs(spec).macs == 8960, "count_macs (acceptance golden)");
  const MacReport r = mac_report(spec, p, 8);
  require(r.original == 8960 && r.dense_folded == 71680 && r.grouped_folded == 8960 && r.zero_padded == 71680 &&
              r.factor == 8,
          "mac_report (acceptance_main.cpp:498-500)");
  require_throws<std::invalid_argument>([&] { mac_report(spec, check_legality(spec, 3, 8), 8); },
                                        "mac_report on a fallback plan");
  return "legality table, count_macs 8960, mac_report 8960/71680/8960/71680";
}

// ---------------------------------------------------------------- device criteria
std::string golden_single_conv() {
  Rng rng(1001);
  const DenseTensor xf = rng.floats({1, 32, 64, 1});
  const DenseTensor wf = rng.floats({5, 1, 1, 1});
  const DenseTensor bf = rng.floats({1});
  const FoldResult rf = apply_width_fold(xf, wf, bf, 8);
  require(rf.plan.ok(), "golden fold must apply");
  const float float_diff = max_abs_diff(pipeline_folded(rf), pipeline_original(xf, wf, bf));
  require(float_diff <= 1e-5f, "float diff above 1e-5");
  const DenseTensor xi = rng.ints({1, 32, 64, 1});
  const DenseTensor wi = rng.ints({5, 1, 1, 1});
  const DenseTensor bi = rng.ints({1});
  const float int_diff = max_abs_diff(pipeline_folded(apply_width_fold(xi, wi, bi, 8)),
                                      pipeline_original(xi, wi, bi));
  require(int_diff == 0.0f, "integer data must match exactly");
  std::ostringstream os;
  os << "float diff " << float_diff << " (tol 1e-5), integer diff " << int_diff;
  return os.str();
}

std::string appendix_a_goldens() {
  if (g_golden.empty()) return "skipped (no golden dir)";
  for (const char* kind : {"float", "int"}) {
    const std::string k(kind);
    const DenseTensor x = load_golden(k + "_x"), w = load_golden(k + "_w"), b = load_golden(k + "_b");
    const FoldResult r = apply_width_fold(x, w, b, 8);
    require(r.plan.ok(), k + ": fold must apply");
    require(r.input.bitwise_equal(load_golden(k + "_x_f")), k + ": x_f differs from the reference's");
    require(r.filter.bitwise_equal(load_golden(k + "_w_f")), k + ": w_f differs from the reference's");
    require(r.bias.bitwise_equal(load_golden(k + "_b_f")), k + ": b_f differs from the reference's");
    require(pipeline_folded(r).bitwise_equal(load_golden(k + "_y_folded")), k + ": folded output differs");
    require(pipeline_original(x, w, b).bitwise_equal(load_golden(k + "_y_ref")), k + ": original output differs");
  }
  return "x_f, w_f, b_f, y_folded, y_ref bitwise equal to the reference's (float + int)";
}

std::string oracle_equivalence_sweep() {
  Rng rng(1002);
  int cases = 0;
  for (const std::int64_t F : {1, 2, 4, 8})
    for (const std::int64_t K : {1, 2, 3})
      for (std::int64_t H = K; H <= 8; ++H)
        for (const std::int64_t W : {F, 2 * F})
          for (const std::int64_t Cout : {1, 2}) {
            const DenseTensor x = rng.ints({1, H, W, 1});
            const DenseTensor w = rng.ints({K, 1, 1, Cout});
            const DenseTensor b = rng.ints({Cout});
            const FoldResult r = apply_width_fold(x, w, b, F);
            require(r.plan.ok(), "sweep case must be legal");
            require(max_abs_diff(pipeline_folded(r), naive_conv_bias(x, w, b)) == 0.0f,
                    "folded result differs from the oracle");
            ++cases;
          }
  require(cases == 336, "sweep size");
  return std::to_string(cases) + " cases exact on integer data";
}

std::string expansion_kats() {
  Rng rng(28);
  const DenseTensor w = rng.floats({5, 1, 1, 1});
  const DenseTensor e = expand_filter(w, 8);
  require(e.shape() == Shape({5, 1, 8, 8}), "expand shape");
  std::int64_t nnz = 0;
  for (std::int64_t k = 0; k < 5; ++k)
    for (std::int64_t f = 0; f < 8; ++f)
      for (std::int64_t fp = 0; fp < 8; ++fp) {
        const float v = e.at({k, 0, f, fp});
        if (f == fp)
          require(v == w.at({k, 0, 0, 0}), "diagonal value");
        else
          require(v == 0.0f && !std::signbit(v), "off-diagonal exact +0.0");
        nnz += v != 0.0f;
      }
  require(nnz == 8 * 5, "exactly F*K*Cout nonzeros");
  require(expand_filter(w, 1).bitwise_equal(w), "factor 1 is the identity");
  const DenseTensor e2 = expand_filter(DenseTensor({1, 1, 1, 2}, {5.0f, 7.0f}), 2);
  require(e2.bitwise_equal(DenseTensor({1, 1, 2, 4}, {5, 7, 0, 0, 0, 0, 5, 7})), "K=1 F=2 Cout=2 block placement");
  require_throws<IllegalFold>([] { expand_filter(DenseTensor::zeros({3, 2, 1, 1}), 2); }, "KW on the fold axis");
  require_throws<IllegalFold>([] { expand_filter(DenseTensor::zeros({3, 1, 2, 1}), 2); }, "Cin != 1");
  const DenseTensor wg = Rng(30).floats({3, 1, 2, 2});
  const DenseTensor eg = expand_filter_general(wg, 3);
  for (std::int64_t k = 0; k < 3; ++k)
    for (std::int64_t ci = 0; ci < 6; ++ci)
      for (std::int64_t co = 0; co < 6; ++co)
        require(eg.at({k, 0, ci, co}) == (ci / 2 == co / 2 ? wg.at({k, 0, ci % 2, co % 2}) : 0.0f),
                "general expansion keeps whole blocks");
  const DenseTensor rb = replicate_bias(DenseTensor({2}, {1.0f, -0.0f}), 3);
  require(rb.bitwise_equal(DenseTensor({6}, {1, -0.0f, 1, -0.0f, 1, -0.0f})), "replicate_bias keeps bits");
  const DenseTensor xg = Rng(31).floats({2, 3, 12, 3});
  for (const std::int64_t F : {1, 2, 3, 4, 6, 12})
    require(unfold_input_general(fold_input_general(xg, F), F).bitwise_equal(xg), "unfold(fold(x)) == x");
  return "expand_filter structure, block placement, general blocks, replicate_bias, fold bijectivity";
}

std::string block_diagonal_and_grouped() {
  Rng rng(40);
  const DenseTensor w = rng.floats({3, 1, 2, 3});
  const DenseTensor wexp = expand_filter_general(w, 4);
  const BlockDiagFilter bd = BlockDiagFilter::from_expanded(wexp, 4);
  require(bd.shared_storage() && bd.num_blocks() == 4, "replicated blocks share storage");
  require(bd.block_shape() == Shape({3, 1, 2, 3}) && bd.logical_shape() == wexp.shape(), "block shapes");
  require(bd.stored_floats() * 4 == wexp.size(), "stored floats = 1/F of the dense expansion");
  require(densify(bd).bitwise_equal(wexp), "densify(from_expanded(w)) == w");
  const DenseTensor x = fold_input_general(rng.floats({2, 7, 16, 2}), 4);
  const ConvSpec spec{x.shape(), wexp.shape()};
  require(grouped_conv(x, bd, spec).bitwise_equal(conv2d(x, wexp, spec)), "grouped == dense conv bitwise");
  std::vector<float> bad(wexp.data().begin(), wexp.data().end());
  bad[3] = 1e-30f;  // (kh=0, cin=0, cout=3): off the diagonal
  require_throws<NotBlockDiagonal>([&] { BlockDiagFilter::from_expanded(DenseTensor(wexp.shape(), bad), 4); },
                                   "strict-zero policy (1e-30)");
  bad[3] = -0.0f;
  (void)BlockDiagFilter::from_expanded(DenseTensor(wexp.shape(), bad), 4);  // -0.0 is a zero
  // a NaN pixel poisons only its own block's outputs on the grouped path
  std::vector<float> xv(x.data().begin(), x.data().end());
  xv[0] = NAN;  // (b=0, h=0, w'=0, channel 0) -> block 0
  const DenseTensor xn(x.shape(), xv);
  const DenseTensor yg = grouped_conv(xn, bd, spec);
  require(std::isnan(yg.at({0, 0, 0, 0})) && !std::isnan(yg.at({0, 0, 0, 3})), "NaN confined to its block");
  std::vector<DenseTensor> blocks;
  for (int g = 0; g < 2; ++g) blocks.push_back(rng.floats({1, 1, 2, 2}));
  const BlockDiagFilter own = BlockDiagFilter::from_blocks(blocks);
  require(!own.shared_storage() && own.densify().at({0, 0, 2, 3}) == blocks[1].at({0, 0, 0, 1}), "from_blocks");
  return "from_expanded / shared / from_blocks / densify, strict zeros, grouped == dense";
}

std::string conv_entry_points() {
  Rng rng(50);
  const DenseTensor x = rng.ints({2, 9, 11, 3});
  const DenseTensor w = rng.ints({3, 2, 3, 5});
  const DenseTensor b = rng.ints({5});
  const ConvSpec spec{x.shape(), w.shape(), 2, 3};
  const DenseTensor y = conv2d(x, w, spec);
  require(y.shape() == spec.output_shape(), "conv2d output shape");
  for (std::int64_t n = 0; n < 2; ++n)
    for (std::int64_t oh = 0; oh < spec.out_h(); ++oh)
      for (std::int64_t ow = 0; ow < spec.out_w(); ++ow)
        for (std::int64_t oc = 0; oc < 5; ++oc) {
          float acc = 0.0f;
          for (std::int64_t kh = 0; kh < 3; ++kh)
            for (std::int64_t kw = 0; kw < 2; ++kw)
              for (std::int64_t ci = 0; ci < 3; ++ci)
                acc += x.at({n, oh * 2 + kh, ow * 3 + kw, ci}) * w.at({kh, kw, ci, oc});
          require(y.at({n, oh, ow, oc}) == acc, "strided conv2d value");
        }
  require(bias_add(y, b).at({1, 1, 1, 4}) == y.at({1, 1, 1, 4}) + b.at({4}), "bias_add");
  require(count_macs(spec).macs == 2ull * 4 * 4 * 5 * 3 * 2 * 3, "count_macs strided");
  const DenseTensor x1 = rng.floats({12, 9, 1});
  const DenseTensor k1 = rng.floats({4});
  const DenseTensor y1 = conv1d_h(x1, k1, 0.5f);
  require(y1.bitwise_equal(reshape(
              bias_add(conv2d(reshape(x1, {1, 12, 9, 1}), reshape(k1, {4, 1, 1, 1}),
                              ConvSpec{{1, 12, 9, 1}, {4, 1, 1, 1}}),
                       DenseTensor({1}, {0.5f})),
              {9, 9, 1})),
          "conv1d_h == conv2d with KW = 1, bitwise");
  require_throws<ShapeMismatch>([&] { conv2d(x, w, ConvSpec{{2, 9, 11, 3}, {3, 2, 3, 4}}); }, "filter vs spec");
  require_throws<ShapeMismatch>([&] { bias_add(y, DenseTensor::zeros({4})); }, "bias length");
  require_throws<ShapeMismatch>([] { conv1d_h(DenseTensor::zeros({3, 4, 1}), DenseTensor::zeros({5}), 0); },
                                "kernel longer than the height");
  return "conv2d (strided, exact), bias_add, conv1d_h, errors";
}

}  // namespace

int main(int argc, char** argv) {
  bool host_only = false;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    if (a == "--host-only")
      host_only = true;
    else
      g_golden = a;
  }
  std::vector<std::pair<std::string, std::function<std::string()>>> criteria = {
      {"values_and_errors", values_and_errors}, {"legality_and_macs", legality_and_macs}};
  if (!host_only) {
    criteria.insert(criteria.end(), {{"golden_single_conv", golden_single_conv},
                                     {"appendix_a_goldens", appendix_a_goldens},
                                     {"oracle_equivalence_sweep", oracle_equivalence_sweep},
                                     {"expansion_kats", expansion_kats},
                                     {"block_diagonal_and_grouped", block_diagonal_and_grouped},
                                     {"conv_entry_points", conv_entry_points}});
  }
  int failures = 0;
  for (const auto& [name, body] : criteria) {
    try {
      const std::string detail = body();
      std::cout << "[PASS] " << name << ": " << detail << "\n";
    } catch (const std::exception& e) {
      ++failures;
      std::cout << "[FAIL] " << name << ": " << e.what() << "\n";
    }
  }
  return failures;
}
