// abi.cpp -- the extern "C" boundary declared in include/widthfold_b200.h.
// Argument validation, plan (re)construction and dispatch to the sm_100a
// launchers. No allocation on the conv path; every call is stream-ordered.
#include <cuda_runtime.h>

#include <atomic>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "kernels.hpp"
#include "plan.hpp"
#include "widthfold_b200.h"

namespace {

thread_local std::string g_last_error;
std::atomic<int> g_num_sms{0};

// Rebuilding a schedule from a plan re-runs the planner (including the
// accumulator-slot order search); forward calls look it up here instead.
// Keyed by the descriptor and the plan bytes; small, thread-safe, bounded.
struct SchedKey {
  wf_conv_desc d;
  wf_fold_plan p;
  bool operator==(const SchedKey& o) const {
    return std::memcmp(&d, &o.d, sizeof(d)) == 0 && std::memcmp(&p, &o.p, sizeof(p)) == 0;
  }
};
// A cached schedule and the launches prepared from it.
struct SchedEntry {
  SchedKey key;
  wfb::Schedule S;
  wfb::LaunchCache launches;
};
std::mutex g_sched_mu;
std::vector<std::shared_ptr<SchedEntry>> g_sched;  // most recently used first
thread_local std::shared_ptr<SchedEntry> t_last;    // this thread's last hit (no lock, no scan)

wf_status cached_schedule(const wf_conv_desc& d, const wf_fold_plan& p, std::shared_ptr<SchedEntry>* out,
                          std::string* err) {
  SchedKey key;
  std::memset(&key, 0, sizeof(key));
  key.d = d;
  key.p = p;
  if (t_last && t_last->key == key) {
    *out = t_last;
    return WF_OK;
  }
  {
    std::lock_guard<std::mutex> lk(g_sched_mu);
    for (size_t i = 0; i < g_sched.size(); ++i)
      if (g_sched[i]->key == key) {
        *out = t_last = g_sched[i];
        if (i) std::swap(g_sched[i], g_sched[0]);
        return WF_OK;
      }
  }
  auto E = std::make_shared<SchedEntry>();
  E->key = key;
  wf_status st = wfb::schedule_from_plan(d, p, &E->S, err);
  if (st != WF_OK) return st;
  std::lock_guard<std::mutex> lk(g_sched_mu);
  g_sched.insert(g_sched.begin(), E);
  if (g_sched.size() > 64) g_sched.pop_back();
  *out = t_last = E;
  return WF_OK;
}

// Epilogue bits wf_conv_fold_fwd accepts: the documented ones, plus the
// 0xFFFF00 profiling switches in a WFB_PROFILE=1 build only.
#ifndef WFB_PROFILE
#define WFB_PROFILE 0
#endif
constexpr uint32_t kEpilogueAccepted =
    WF_EPI_BIAS | WF_EPI_RELU | WF_EPI_PREPITCHED | WF_EPI_ROW_PRODUCER | (WFB_PROFILE ? 0xFFFF00u : 0u);

wf_status fail(wf_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

}  // namespace

extern "C" {

int wf_abi_version(void) { return 6; }

const char* wf_last_error(void) { return g_last_error.c_str(); }

void wf_set_num_sms(int num_sms) { g_num_sms.store(num_sms < 0 ? 0 : num_sms); }

wf_status wf_plan_fold(const wf_conv_desc* desc, int64_t f, int64_t group_size, wf_dtype in_dtype,
                       wf_fold_plan* plan) {
  if (!desc || !plan) return fail(WF_INVALID_ARGUMENT, "null argument");
  wfb::Schedule S;
  std::string err;
  wf_status st = wfb::make_schedule(*desc, f, group_size, in_dtype, &S, &err);
  if (st != WF_OK) return fail(st, err);
  *plan = S.plan;
  return WF_OK;
}

wf_status wf_plan_unfolded(const wf_conv_desc* desc, wf_dtype in_dtype, wf_fold_plan* plan) {
  if (!desc || !plan) return fail(WF_INVALID_ARGUMENT, "null argument");
  wfb::Schedule S;
  std::string err;
  wf_status st = wfb::make_schedule_unfolded(*desc, in_dtype, &S, &err);
  if (st != WF_OK) return fail(st, err);
  *plan = S.plan;
  return WF_OK;
}

wf_status wf_schedule_describe(const wf_conv_desc* desc, int64_t f, int64_t group_size, wf_dtype in_dtype,
                               char* buf, size_t cap) {
  if (!desc || !buf) return fail(WF_INVALID_ARGUMENT, "null argument");
  wfb::Schedule S;
  std::string err;
  wf_status st = wfb::make_schedule(*desc, f, group_size, in_dtype, &S, &err);
  if (st != WF_OK) return fail(st, err);
  if (S.plan.status != WF_FOLD_APPLY) return fail(WF_INVALID_ARGUMENT, "plan falls back: nothing to describe");
  std::string j = "{";
  auto kv = [&](const char* k, long long v) { j += "\"" + std::string(k) + "\": " + std::to_string(v) + ", "; };
  auto arr = [&](const char* k, const std::vector<long long>& v) {
    j += "\"" + std::string(k) + "\": [";
    for (size_t i = 0; i < v.size(); ++i) j += (i ? ", " : "") + std::to_string(v[i]);
    j += "], ";
  };
  kv("f", S.plan.f); kv("r", S.plan.r); kv("c0", S.plan.c0); kv("kw_f", S.plan.kw_f); kv("s", S.s);
  kv("ph", S.ph); kv("pw", S.pw); kv("esize", S.esize); kv("Q", S.Q); kv("Ng", S.Ng); kv("CH", S.CH);
  kv("wbox", S.plan.wbox); kv("tile_rows", S.plan.tile_rows); kv("nrows", S.plan.nrows); kv("tps", S.tps);
  kv("tile_shift", S.tile_shift); kv("sw32", S.sw32); kv("kpair", S.kpair); kv("need_shift", S.need_shift);
  kv("region_bytes", S.region_bytes); kv("qregion_bytes", S.qregion_bytes); kv("lbo_a", S.lbo_a);
  kv("stage_bytes", S.stage_bytes); kv("stages", S.stages); kv("smem_bytes", S.smem_bytes);
  std::vector<long long> v;
  for (int b = 0; b < S.s; ++b) v.push_back(S.has_res[b] ? S.amin[b] : -999);
  arr("amin", v);
  arr("qs", std::vector<long long>(S.qs.begin(), S.qs.end()));
  arr("order", std::vector<long long>(S.order.begin(), S.order.end()));
  v.clear();
  for (const auto& t : S.ntiles) { v.push_back(t.col0); v.push_back(t.cols); v.push_back(t.entry0); v.push_back(t.entries); v.push_back(t.g0); v.push_back(t.split); }
  arr("ntiles", v);
  v.clear();
  for (size_t i = 0; i < S.entries.size(); ++i) {
    const auto& e = S.entries[i];
    v.push_back(e.a_off); v.push_back(S.entry_lbo[i]); v.push_back(e.b_off); v.push_back(e.meta);
    v.push_back(e.tmem_col); v.push_back(S.entry_cc0[i]); v.push_back(S.entry_cc1[i]);
  }
  arr("entries", v);
  j += "\"mma_entries\": " + std::to_string(S.entries.size()) + "}";
  if (j.size() + 1 > cap) return fail(WF_INVALID_ARGUMENT, "buffer too small: need " + std::to_string(j.size() + 1));
  std::memcpy(buf, j.c_str(), j.size() + 1);
  return WF_OK;
}

size_t wf_packed_filter_bytes(const wf_fold_plan* plan) {
  if (!plan || plan->status != WF_FOLD_APPLY) return 0;
  return static_cast<size_t>(plan->packed_bytes);
}

wf_status wf_expand_filter_pack(const void* w, const float* b, const wf_conv_desc* desc, const wf_fold_plan* plan,
                                void* w_packed, float* b_rep, void* stream) {
  if (!w || !desc || !plan || !w_packed) return fail(WF_INVALID_ARGUMENT, "null argument");
  wfb::Schedule S;
  std::string err;
  wf_status st = wfb::schedule_from_plan(*desc, *plan, &S, &err);
  if (st != WF_OK) return fail(st, err);
  st = wfb::launch_pack(S, *desc, w, b, w_packed, b_rep, static_cast<cudaStream_t>(stream), &err);
  if (st != WF_OK) return fail(st, err);
  return WF_OK;
}

wf_status wf_expand_filter_dense(const float* w, const wf_conv_desc* desc, int64_t f, float* w_dense, void* stream) {
  if (!w || !desc || !w_dense) return fail(WF_INVALID_ARGUMENT, "null argument");
  std::string err;
  wf_status st = wfb::validate_desc(*desc, &err);
  if (st != WF_OK) return fail(st, err);
  if (f < 1) return fail(WF_INVALID_ARGUMENT, "fold factor must be >= 1");
  if (f % desc->stride_w != 0) return fail(WF_ILLEGAL_FOLD, "fold factor must be a multiple of stride_w");
  st = wfb::launch_expand_dense(*desc, f, w, w_dense, static_cast<cudaStream_t>(stream), &err);
  if (st != WF_OK) return fail(st, err);
  return WF_OK;
}

wf_status wf_conv_fold_fwd_ws(const void* x, void* workspace, const void* w_packed, const float* b_rep, void* y,
                              const wf_conv_desc* desc, const wf_fold_plan* plan, wf_dtype out_dtype,
                              uint32_t epilogue, void* stream) {
  if (!x || !w_packed || !y || !desc || !plan) return fail(WF_INVALID_ARGUMENT, "null argument");
  if (epilogue & ~kEpilogueAccepted) return fail(WF_INVALID_ARGUMENT, "unknown epilogue flags");
  if (plan->workspace_bytes > 0 && !workspace && !(epilogue & WF_EPI_ROW_PRODUCER))
    return fail(WF_INVALID_ARGUMENT, "this plan needs a workspace of plan->workspace_bytes (wf_conv_fold_fwd_ws)");
  std::shared_ptr<SchedEntry> E;
  std::string err;
  wf_status st = cached_schedule(*desc, *plan, &E, &err);
  if (st != WF_OK) return fail(st, err);
  st = wfb::launch_conv(E->S, *desc, x, workspace, w_packed, b_rep, y, out_dtype, epilogue,
                        static_cast<cudaStream_t>(stream), g_num_sms.load(), &E->launches, &err);
  if (st != WF_OK) return fail(st, err);
  return WF_OK;
}

wf_status wf_conv_fold_fwd(const void* x, const void* w_packed, const float* b_rep, void* y,
                           const wf_conv_desc* desc, const wf_fold_plan* plan, wf_dtype out_dtype, uint32_t epilogue,
                           void* stream) {
  return wf_conv_fold_fwd_ws(x, nullptr, w_packed, b_rep, y, desc, plan, out_dtype, epilogue, stream);
}

wf_status wf_repitch_input(const void* x, void* workspace, const wf_conv_desc* desc, const wf_fold_plan* plan,
                           void* stream) {
  if (!x || !desc || !plan) return fail(WF_INVALID_ARGUMENT, "null argument");
  if (plan->workspace_bytes == 0 || plan->producer != 3) return WF_OK;
  if (!workspace) return fail(WF_INVALID_ARGUMENT, "this plan needs a workspace of plan->workspace_bytes");
  std::shared_ptr<SchedEntry> E;
  std::string err;
  wf_status st = cached_schedule(*desc, *plan, &E, &err);
  if (st != WF_OK) return fail(st, err);
  st = wfb::launch_repitch_input(E->S, *desc, x, workspace, static_cast<cudaStream_t>(stream), &err);
  if (st != WF_OK) return fail(st, err);
  return WF_OK;
}

wf_status wf_conv_direct_fwd(const float* x, const float* w, float* y, const wf_conv_desc* desc, void* stream) {
  if (!x || !w || !y || !desc) return fail(WF_INVALID_ARGUMENT, "null argument");
  std::string err;
  wf_status st = wfb::validate_desc(*desc, &err);
  if (st != WF_OK) return fail(st, err);
  st = wfb::launch_conv_direct(*desc, x, w, y, 1, static_cast<cudaStream_t>(stream), &err);
  if (st != WF_OK) return fail(st, err);
  return WF_OK;
}

wf_status wf_conv_grouped_fwd(const float* x, const float* w_dense, float* y, const wf_conv_desc* desc,
                              int64_t groups, void* stream) {
  if (!x || !w_dense || !y || !desc) return fail(WF_INVALID_ARGUMENT, "null argument");
  std::string err;
  wf_status st = wfb::validate_desc(*desc, &err);
  if (st != WF_OK) return fail(st, err);
  if (groups < 1 || desc->c % groups != 0 || desc->cout % groups != 0)
    return fail(WF_SHAPE_MISMATCH, "channel extents not divisible into the requested groups");
  st = wfb::launch_conv_direct(*desc, x, w_dense, y, static_cast<int>(groups), static_cast<cudaStream_t>(stream),
                               &err);
  if (st != WF_OK) return fail(st, err);
  return WF_OK;
}

wf_status wf_cast_f32(const float* x, void* y, int64_t n, wf_dtype to, void* stream) {
  if ((!x || !y) && n > 0) return fail(WF_INVALID_ARGUMENT, "null argument");
  if (n <= 0) return WF_OK;
  std::string err;
  wf_status st = wfb::launch_cast_f32(x, y, n, to, static_cast<cudaStream_t>(stream), &err);
  if (st != WF_OK) return fail(st, err);
  return WF_OK;
}

wf_status wf_bias_add(const float* y, const float* b, float* out, int64_t n, int64_t c, int32_t relu, void* stream) {
  if (!y || !b || !out) return fail(WF_INVALID_ARGUMENT, "null argument");
  if (c < 1 || n < 0 || n % c != 0) return fail(WF_SHAPE_MISMATCH, "bias length does not divide the output");
  std::string err;
  wf_status st = wfb::launch_bias_add(y, b, out, n, static_cast<int>(c), relu, static_cast<cudaStream_t>(stream), &err);
  if (st != WF_OK) return fail(st, err);
  return WF_OK;
}

wf_status wf_replicate_bias(const float* b, int64_t cout, int64_t r, float* out, void* stream) {
  if (!b || !out) return fail(WF_INVALID_ARGUMENT, "null argument");
  if (r < 1) return fail(WF_INVALID_ARGUMENT, "fold factor must be >= 1");
  if (cout < 1) return fail(WF_SHAPE_MISMATCH, "bias must be non-empty");
  std::string err;
  wf_status st = wfb::launch_replicate_bias(b, static_cast<int>(cout), static_cast<int>(r), out,
                                            static_cast<cudaStream_t>(stream), &err);
  if (st != WF_OK) return fail(st, err);
  return WF_OK;
}

wf_status wf_check_block_diagonal(const float* w_dense, int64_t kh, int64_t kw, int64_t cif, int64_t cof,
                                  int64_t groups, void* scratch, int64_t* first_bad, void* stream) {
  if (!w_dense || !scratch || !first_bad) return fail(WF_INVALID_ARGUMENT, "null argument");
  if (groups < 1 || cif % groups != 0 || cof % groups != 0)
    return fail(WF_SHAPE_MISMATCH, "channel extents not divisible into the requested blocks");
  std::string err;
  long long bad = -1;
  wf_status st = wfb::launch_blockdiag_check(w_dense, static_cast<int>(kh), static_cast<int>(kw),
                                             static_cast<int>(cif), static_cast<int>(cof), static_cast<int>(groups),
                                             static_cast<unsigned long long*>(scratch), &bad,
                                             static_cast<cudaStream_t>(stream), &err);
  if (st != WF_OK) return fail(st, err);
  *first_bad = bad;
  if (bad >= 0) return fail(WF_NOT_BLOCK_DIAGONAL, "off-diagonal entry at flat index " + std::to_string(bad) + " is nonzero");
  return WF_OK;
}

}  // extern "C"
