// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A thin extern "C" face over the UNMODIFIED reference library compiled from
// /root/reference/proj/src (see oracle/Makefile). It lets tests/ and bench.py's
// reference arm call the reference's own CPU conv path through ctypes:
//   widthfold::conv2d      /root/reference/proj/src/refconv.cpp:34-80
//   widthfold::bias_add    /root/reference/proj/src/refconv.cpp:82-95
//   widthfold::expand_filter_general  /root/reference/proj/src/fold.cpp:185-211
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
// reference) may load the resulting oracle/_ref/libwidthfold_ref.so.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "widthfold/fold.hpp"
#include "widthfold/refconv.hpp"

namespace wf = widthfold;

namespace {
thread_local std::string g_err;
wf::DenseTensor make(const float* p, wf::Shape s) {
  std::vector<float> d(static_cast<std::size_t>(wf::numel(s)));
  std::memcpy(d.data(), p, d.size() * sizeof(float));
  return wf::DenseTensor(std::move(s), std::move(d));
}
}  // namespace

extern "C" {

const char* wfref_last_error(void) { return g_err.c_str(); }

// y = conv2d(x, w, stride) [+ bias_add(b)] [relu] on one VALID problem.
// relu is NOT a reference operation (the reference has none); it is applied
// after bias_add exactly as the B200 epilogue does, for the MNv2 config.
int wfref_conv2d(const float* x, int64_t B, int64_t H, int64_t W, int64_t C,
                 const float* w, int64_t KH, int64_t KW, int64_t Cout,
                 int64_t sh, int64_t sw, const float* b, int relu, float* y) {
  try {
    const wf::DenseTensor xt = make(x, {B, H, W, C});
    const wf::DenseTensor wt = make(w, {KH, KW, C, Cout});
    const wf::ConvSpec spec{xt.shape(), wt.shape(), sh, sw};
    wf::DenseTensor out = wf::conv2d(xt, wt, spec);
    if (b) out = wf::bias_add(out, make(b, {Cout}));
    const auto d = out.data();
    for (std::size_t i = 0; i < d.size(); ++i) {
      float v = d[i];
      if (relu && !(v > 0.0f)) v = (v != v) ? v : 0.0f;
      y[i] = v;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int wfref_expand_filter_general(const float* w, int64_t KH, int64_t KW,
                                int64_t C, int64_t Cout, int64_t factor,
                                float* out) {
  try {
    const wf::DenseTensor e =
        wf::expand_filter_general(make(w, {KH, KW, C, Cout}), factor);
    std::memcpy(out, e.data().data(), e.data().size() * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // extern "C"
