// plan.cpp -- see plan.hpp for the geometry and the schedule it produces.
#include "plan.hpp"

#include <algorithm>
#include <functional>
#include <cstdlib>
#include <numeric>

namespace wfb {

namespace {
// Producer request for unaligned rows of the planner call on this thread:
// -1 the default (WF_GATHER=1 overrides it), 3 / 4 forced (schedule_from_plan
// rebuilds a plan with its own producer).
thread_local int g_prod_req = -1;
struct ProdScope {
  int saved;
  explicit ProdScope(int v) : saved(g_prod_req) { g_prod_req = v; }
  ~ProdScope() { g_prod_req = saved; }
};
}  // namespace

namespace {

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
int64_t floor_div(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}
int64_t pos_mod(int64_t a, int64_t b) { return ((a % b) + b) % b; }

wf_fold_plan fallback(wf_fold_reason reason, int64_t f) {
  wf_fold_plan p{};
  p.status = WF_FOLD_FALLBACK;
  p.reason = reason;
  p.f = f;
  return p;
}

}  // namespace

int elem_bytes(wf_dtype t) {
  switch (t) {
    case WF_BF16: case WF_F16: return 2;
    case WF_TF32: case WF_F32: return 4;
  }
  return 0;
}

wf_status validate_desc(const wf_conv_desc& d, std::string* err) {
  const int64_t ext[7] = {d.n, d.h, d.w, d.c, d.kh, d.kw, d.cout};
  for (int64_t e : ext) {
    if (e < 1) {
      *err = "conv extents must be >= 1";
      return WF_SHAPE_MISMATCH;
    }
  }
  if (d.stride_h < 1 || d.stride_w < 1) {
    *err = "strides must be >= 1";
    return WF_SHAPE_MISMATCH;
  }
  if (d.pad_h < 0 || d.pad_w < 0) {
    *err = "padding must be >= 0";
    return WF_SHAPE_MISMATCH;
  }
  if (d.h + 2 * d.pad_h < d.kh || d.w + 2 * d.pad_w < d.kw) {
    *err = "padded input smaller than the filter: empty output";
    return WF_DEGENERATE_OUTPUT;
  }
  return WF_OK;
}

namespace {
wf_status make_schedule_tps(const wf_conv_desc& d, int64_t f_req, int64_t gs_req, wf_dtype in_dtype, int tps,
                            Schedule* out, std::string* err, int kpair_req = -1, int pair_req = 0);

int64_t mma_cost(int64_t n) { return std::max<int64_t>(n / 2, 32 + n / 4); }

// One kpair MMA: accumulator slots [slot0, slot0 + len) of the N-tile; core
// column k in {0, 1} is (kh[k], c[k]) and feeds the slots in mask[k] (bit i =
// slot slot0 + i; the other rows of its B half-block are zero).
struct PMma {
  int slot0, len;
  int kh[2], c[2];
  uint32_t mask[2];
};

// kpair MMAs of one N-tile. ord[slot] = group; group g's window covers core
// columns [lo[g], hi[g]] of every kh row. Items (kh, c) with the same
// accumulator run pair up among themselves ((c, kh) order: mostly (kh, c) with
// (kh+1, c)); the odd ones out are matched by a min-cost DP over their runs'
// hulls, a last single one pairs with a zero (mask 0) neighbour column.
std::vector<PMma> build_kpair(const std::vector<int>& ord, const std::vector<int64_t>& lo,
                              const std::vector<int64_t>& hi, int KH, int Ng, int64_t max_col) {
  const int ns = static_cast<int>(ord.size());
  int64_t cmin = INT64_MAX, cmax = -1;
  for (int g : ord) { cmin = std::min(cmin, lo[g]); cmax = std::max(cmax, hi[g]); }
  struct Run { int s0, len; };
  std::vector<std::pair<Run, std::vector<std::pair<int, int>>>> groups;  // run -> items (kh, c)
  for (int64_t c = cmin; c <= cmax; ++c) {
    for (int s = 0; s < ns;) {
      if (!(lo[ord[s]] <= c && c <= hi[ord[s]])) { ++s; continue; }
      int e = s;
      while (e < ns && lo[ord[e]] <= c && c <= hi[ord[e]]) ++e;
      size_t k = 0;
      while (k < groups.size() && !(groups[k].first.s0 == s && groups[k].first.len == e - s)) ++k;
      if (k == groups.size()) groups.push_back({Run{s, e - s}, {}});
      for (int kh = 0; kh < KH; ++kh) groups[k].second.push_back({kh, static_cast<int>(c)});
      s = e;
    }
  }
  std::vector<PMma> out;
  struct Left { Run run; int kh, c; };
  std::vector<Left> left;
  for (auto& gr : groups) {
    auto& it = gr.second;
    std::sort(it.begin(), it.end(), [](const std::pair<int, int>& x, const std::pair<int, int>& y) {
      return x.second != y.second ? x.second < y.second : x.first < y.first;
    });
    const uint32_t full = (1u << gr.first.len) - 1u;
    size_t i = 0;
    for (; i + 1 < it.size(); i += 2)
      out.push_back({gr.first.s0, gr.first.len, {it[i].first, it[i + 1].first}, {it[i].second, it[i + 1].second},
                     {full, full}});
    if (i < it.size()) left.push_back({gr.first, it[i].first, it[i].second});
  }
  // leftovers: min-cost matching (hull of the two runs) by DP over subsets
  const int L = static_cast<int>(left.size());
  auto hull_cost = [&](int i, int j) {
    const int a0 = std::min(left[i].run.s0, left[j].run.s0);
    const int a1 = std::max(left[i].run.s0 + left[i].run.len, left[j].run.s0 + left[j].run.len);
    return mma_cost(static_cast<int64_t>(a1 - a0) * Ng);
  };
  std::vector<std::pair<int, int>> match;  // (i, j), j == -1: paired with a zero column
  if (L <= 16) {
    std::vector<int64_t> best(static_cast<size_t>(1) << L, INT64_MAX);
    std::vector<int> pick(static_cast<size_t>(1) << L, -2);
    best[0] = 0;
    for (uint32_t m = 1; m < (1u << L); ++m) {
      const int i = __builtin_ctz(m);
      const uint32_t r = m & ~(1u << i);
      if (best[r] != INT64_MAX) {
        const int64_t c = best[r] + mma_cost(static_cast<int64_t>(left[i].run.len) * Ng);
        if (c < best[m]) { best[m] = c; pick[m] = -1; }
      }
      for (int j = i + 1; j < L; ++j) {
        if (!((r >> j) & 1u) || best[r & ~(1u << j)] == INT64_MAX) continue;
        const int64_t c = best[r & ~(1u << j)] + hull_cost(i, j);
        if (c < best[m]) { best[m] = c; pick[m] = j; }
      }
    }
    for (uint32_t m = (1u << L) - 1u; m;) {
      const int i = __builtin_ctz(m);
      const int j = pick[m];
      match.push_back({i, j});
      m &= ~(1u << i);
      if (j >= 0) m &= ~(1u << j);
    }
  } else {
    int i = 0;
    for (; i + 1 < L; i += 2) match.push_back({i, i + 1});
    if (i < L) match.push_back({i, -1});
  }
  for (const auto& pr : match) {
    const Left& x = left[pr.first];
    if (pr.second < 0) {
      // partner: a neighbouring core column of the same window row (loaded,
      // finite data) with zero B rows; a one-column window row pairs the
      // column with itself (LBO 0) -- a column outside the window could read
      // past the loaded A rows, and 0 * NaN from unloaded shared memory is NaN
      const int c2 = x.c > 0 ? x.c - 1 : (x.c + 1 <= max_col ? x.c + 1 : x.c);
      out.push_back({x.run.s0, x.run.len, {x.kh, x.kh}, {x.c, c2}, {(1u << x.run.len) - 1u, 0u}});
      continue;
    }
    const Left& y = left[pr.second];
    const int s0 = std::min(x.run.s0, y.run.s0);
    const int s1 = std::max(x.run.s0 + x.run.len, y.run.s0 + y.run.len);
    out.push_back({s0, s1 - s0, {x.kh, y.kh}, {x.c, y.c},
                   {((1u << x.run.len) - 1u) << (x.run.s0 - s0), ((1u << y.run.len) - 1u) << (y.run.s0 - s0)}});
  }
  return out;
}

// Order runs (slot0, len) so each one meets only untouched accumulator slots
// (its MMA zero-initialises them) or only touched ones. Backtracking, widest
// first; false when no such order exists.
bool zero_init_order(const std::vector<std::pair<int, int>>& runs, int nslots, std::vector<int>* seq_out) {
  std::vector<int> idx(runs.size());
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return runs[x].second > runs[y].second; });
  std::vector<char> used(runs.size(), 0), tch(static_cast<size_t>(nslots), 0);
  std::vector<int> seq;
  int budget = 100000;
  std::function<bool()> place = [&]() -> bool {
    if (seq.size() == runs.size()) return true;
    if (--budget < 0) return false;
    for (int k : idx) {
      if (used[k]) continue;
      int nt = 0;
      for (int q = 0; q < runs[k].second; ++q) nt += tch[runs[k].first + q];
      if (nt != 0 && nt != runs[k].second) continue;
      std::vector<char> saved = tch;
      for (int q = 0; q < runs[k].second; ++q) tch[runs[k].first + q] = 1;
      used[k] = 1;
      seq.push_back(k);
      if (place()) return true;
      seq.pop_back();
      used[k] = 0;
      tch = saved;
      if (nt != 0) break;  // an all-touched run fits anywhere: no other choice is better here
    }
    return false;
  };
  if (!place()) return false;
  *seq_out = seq;
  return true;
}
}  // namespace

// Variant selection over one planner core (make_schedule_tps):
//  * CTA pairs (cta_group::2, each SM holding half of every B block, so a B
//    that needs two N-tiles on one CTA fits in one) only on request
//    (WF_CTA_PAIR=1): measured slower on B200 even for AlexNet (B = 173 KB,
//    0.290 vs 0.278 ms with two N-tiles);
//  * else two M tiles per A stage (their input-row halo loaded once) when it
//    fits as well as one tile per stage does and the batch is large; WF_TPS=1
//    forces one.
// kpair_req / pair_req / tps_req >= 0 pin a choice (schedule_from_plan).
static wf_status make_schedule_variant(const wf_conv_desc& d, int64_t f_req, int64_t gs_req, wf_dtype in_dtype,
                                       Schedule* out, std::string* err, int kpair_req, int pair_req, int tps_req) {
  if (pair_req < 0) {
    const char* env = std::getenv("WF_CTA_PAIR");
    if (env && (env[0] == '0' || env[0] == '1')) pair_req = env[0] - '0';
  }
  if (f_req == 0) return make_schedule_tps(d, f_req, gs_req, in_dtype, 1, out, err, kpair_req, pair_req < 0 ? -1 : pair_req);
  if (pair_req == 1) return make_schedule_tps(d, f_req, gs_req, in_dtype, 1, out, err, kpair_req, 1);
  Schedule s1;
  wf_status st = make_schedule_tps(d, f_req, gs_req, in_dtype, 1, &s1, err, kpair_req, 0);
  if (st == WF_OK && s1.plan.status != WF_FOLD_APPLY && s1.plan.reason == WF_REASON_NOT_PROFITABLE &&
      pair_req < 0) {
    // B too large for one SM's shared memory: CTA pairs hold half of it each
    // (e.g. AlexNet zero-padded to Cin = 8, B = 270 KB)
    Schedule sp;
    std::string e2;
    if (make_schedule_tps(d, f_req, gs_req, in_dtype, 1, &sp, &e2, kpair_req, 1) == WF_OK &&
        sp.plan.status == WF_FOLD_APPLY && sp.pair == 2) {
      *out = std::move(sp);
      return WF_OK;
    }
  }
  if (st != WF_OK || s1.plan.status != WF_FOLD_APPLY) {
    *out = std::move(s1);
    return st;
  }
  // M tiles per A stage: 2 when the stage still double-buffers, the N-tiling
  // is unchanged and every SM keeps >= 4 stage units (small batches keep their
  // parallelism); WF_TPS=1/2/4 forces one. 4 is supported but measured 1-3%
  // slower than 2 (R50, MNv2, VGG): fewer halo rows, shallower pipeline.
  const char* env = std::getenv("WF_TPS");
  const int env_tps = (env && (env[0] == '1' || env[0] == '2' || env[0] == '4')) ? env[0] - '0' : 0;
  for (int cand : {4, 2}) {
    const bool want = (tps_req > 0) ? tps_req == cand
                                    : (env_tps ? env_tps == cand
                                               : cand == 2 && s1.ohb >= cand && d.n * ceil_div(s1.ohb, cand) >= 4 * 148 &&
                                                     d.stride_h > 1);  // H stride 1 (VGG): one tile per stage measured faster
    if (!want || !(s1.prod == 0 || s1.prod >= 3) || s1.pair != 1) continue;
    Schedule s2;
    std::string e2;
    if (make_schedule_tps(d, f_req, gs_req, in_dtype, cand, &s2, &e2, kpair_req, 0) == WF_OK &&
        s2.plan.status == WF_FOLD_APPLY && s2.stages >= 2 && s2.ntiles.size() == s1.ntiles.size() &&
        s2.prod == s1.prod) {
      *out = std::move(s2);
      return WF_OK;
    }
  }
  *out = std::move(s1);
  return WF_OK;
}

namespace {
wf_status make_schedule_tps(const wf_conv_desc& d, int64_t f_req, int64_t gs_req, wf_dtype in_dtype, int tps,
                            Schedule* out, std::string* err, int kpair_req, int pair_req) {
  wf_status st = validate_desc(d, err);
  if (st != WF_OK) return st;
  if (in_dtype != WF_BF16 && in_dtype != WF_F16 && in_dtype != WF_TF32) {
    *err = "input dtype must be bf16, f16 or tf32";
    return WF_INVALID_ARGUMENT;
  }
  if (f_req < 0 || gs_req < 0) {
    *err = "fold factor / group size must be >= 0 (0 = auto)";
    return WF_INVALID_ARGUMENT;
  }
  Schedule S;
  S.esize = elem_bytes(in_dtype);
  S.E = 32 / S.esize;
  const int64_t sh = d.stride_h, sw = d.stride_w;
  S.s = static_cast<int>(sh);
  S.ph = static_cast<int>(d.pad_h);
  S.pw = static_cast<int>(d.pad_w);
  const int64_t OH = (d.h + 2 * d.pad_h - d.kh) / sh + 1;
  const int64_t OW = (d.w + 2 * d.pad_w - d.kw) / sw + 1;

  // ---- fold factor ------------------------------------------------------
  int64_t f = f_req;
  if (f == 0) {
    // smallest f: multiple of the W stride, 16-byte folded pixel, divides W,
    // r*Cout groupable (the auto rule of choose_fold_factor, src/fold.cpp:67-90,
    // with the tcgen05 K-step as the alignment target).
    const int64_t pix = d.c * S.esize;
    const int64_t base_align = 16 / std::gcd<int64_t>(pix, 16);
    const int64_t base = std::lcm<int64_t>(base_align, sw);
    wf_fold_plan first{};
    bool have = false;
    // no factor past 255 core columns per folded pixel can plan (the Q + 1 <= 256
    // limit below), so the search is bounded whatever W is
    const int64_t f_max = std::min<int64_t>(d.w, 255 * 16 / std::max<int64_t>(pix, 1));
    for (int64_t cand = base; cand <= f_max; cand += base) {
      Schedule tmp;
      std::string e2;
      wf_status s2 = make_schedule(d, cand, gs_req, in_dtype, &tmp, &e2, kpair_req, pair_req);
      if (s2 != WF_OK) {
        *err = e2;
        return s2;
      }
      if (tmp.plan.status == WF_FOLD_APPLY) {
        *out = std::move(tmp);
        return WF_OK;
      }
      if (!have) {
        first = tmp.plan;
        have = true;
      }
    }
    S.plan = have ? first : fallback(WF_REASON_FACTOR_TOO_LARGE, base);
    *out = std::move(S);
    return WF_OK;
  }
  if (f % sw != 0) { S.plan = fallback(WF_REASON_STRIDE_ON_FOLD_AXIS, f); *out = S; return WF_OK; }
  if ((f * d.c * S.esize) % 16 != 0) { S.plan = fallback(WF_REASON_UNALIGNED_PIXEL, f); *out = S; return WF_OK; }
  const int64_t r = f / sw;
  if (d.h < sh) { S.plan = fallback(WF_REASON_NOT_PROFITABLE, f); *out = S; return WF_OK; }

  const int64_t c0 = -ceil_div(d.pad_w, f);
  const int64_t kwf = floor_div(f - sw - d.pad_w + d.kw - 1, f) - c0 + 1;
  // W % f != 0: the last folded pixel is partial (zero-filled by the gather
  // producer); OW % r != 0: the last folded output column is masked per j.
  int64_t Wf = ceil_div(d.w, f);
  const int64_t Wfo = ceil_div(OW, r);
  // TMA boxes need the folded view to be a pure reshape with a 16-byte row
  // pitch (and a box must start 16-byte aligned: an element-granular view of
  // x faults on B200, tools/probes/tma_elem_probe.cu). When W % f != 0 or the
  // row pitch is not a 16-byte multiple (AlexNet: W=227, 1362-byte rows):
  //  3 (default) re-pitch x into a workspace of Wp columns (Wp % f == 0,
  //    16-byte rows, zero tail), then the 5-D TMA boxes;
  //  4 (WF_GATHER=1) rows staged in shared memory and realigned by gather
  //    warps -- no workspace, but measured 1.13-1.16x slower than 3.
  int64_t Wp = d.w;
  while (Wp % f != 0 || (Wp * d.c * S.esize) % 16 != 0) ++Wp;
  S.Wp = Wp;
  S.prod = (Wp == d.w) ? 0 : 3;
  Wf = Wp / f;
  const int64_t Q = f * d.c * S.esize / 16;  // core columns per folded pixel
  S.Q = static_cast<int>(Q);
  const int64_t E2 = S.E / 2;                  // elements per core column
  // Folded columns per output row in the A layout: >= Wfo + KW' - 1 and a
  // divisor or multiple of 32, so each epilogue warp (32 TMEM lanes) owns whole
  // output rows (Wbox <= 32) or a 32-column slice of one (Wbox >= 32).
  int64_t Wbox = 1;
  while (Wbox < Wfo + kwf - 1) Wbox *= 2;
  if (Wbox > kTileM || Q + 1 > 256) { S.plan = fallback(WF_REASON_NOT_PROFITABLE, f); *out = S; return WF_OK; }
  // Never shrunk to OH: rows past OH are zero-filled on load and clipped on store.
  const int64_t OHt = kTileM / Wbox;

  // ---- residues of the H stride -----------------------------------------
  if (sh > kMaxResidues) { S.plan = fallback(WF_REASON_NOT_PROFITABLE, f); *out = S; return WF_OK; }
  for (int b = 0; b < sh; ++b) { S.has_res[b] = false; S.amin[b] = 0; S.amax[b] = 0; }
  for (int64_t kh = 0; kh < d.kh; ++kh) {
    const int64_t delta = kh - d.pad_h;
    const int b = static_cast<int>(pos_mod(delta, sh));
    const int a = static_cast<int>((delta - b) / sh);
    if (!S.has_res[b]) { S.has_res[b] = true; S.amin[b] = a; S.amax[b] = a; }
    S.amin[b] = std::min(S.amin[b], a);
    S.amax[b] = std::max(S.amax[b], a);
  }
  S.tps = tps;
  int64_t NR = 0;  // input rows per residue region: tps tiles of OHt output rows + the kh spread
  for (int b = 0; b < sh; ++b)
    if (S.has_res[b]) NR = std::max<int64_t>(NR, tps * OHt + S.amax[b] - S.amin[b]);
  // every core-column region (and the shifted one) must start 128-byte aligned
  // for the TMA destination: pad rows so NR*Wbox*16 % 128 == 0
  while ((NR * Wbox) % 8 != 0) ++NR;
  if (NR > 256) { S.plan = fallback(WF_REASON_NOT_PROFITABLE, f); *out = S; return WF_OK; }
  if (S.prod == 3) {
    int64_t rows = 0;  // raw rows per stage unit (the row table holds <= 64)
    for (int b = 0; b < sh; ++b)
      if (S.has_res[b]) rows += S.amax[b] - S.amin[b] + tps * OHt;
    int want = g_prod_req;
    if (want < 0) {
      const char* eg = std::getenv("WF_GATHER");
      const char* er = std::getenv("WF_REPITCH");
      const char* eq = std::getenv("WF_RING");
      want = (eg && eg[0] == '1') ? 4 : ((eg && eg[0] == '2') ? 6 : ((eq && eq[0] == '1') ? 5 : 3));
      (void)er;
    }
    // 4: 16-bit data, <= 128 row blocks, single-CTA plans
    if ((want == 4 || want == 6) && in_dtype != WF_TF32 && S.esize == 2 && Q * Wbox + 2 <= 128 && rows <= 64 &&
        pair_req != 1)
      S.prod = static_cast<int>(want);  // 6: the same gather warps loading the rows straight from x (L2-prefetched)
    // 5: 16-bit data, a re-pitched row of <= 127 16-byte blocks (4 per gather lane), single-CTA plans
    if (want == 5 && in_dtype != WF_TF32 && (Wp * d.c * S.esize) / 16 + 1 <= 128 && pair_req != 1) {
      int amin_min = INT32_MAX, amax_max = INT32_MIN;
      for (int b = 0; b < sh; ++b)
        if (S.has_res[b]) { amin_min = std::min(amin_min, S.amin[b]); amax_max = std::max(amax_max, S.amax[b]); }
      S.prod = 5;
      S.amin_min = amin_min;
      S.ring_rows = static_cast<int>((amax_max - amin_min + tps * OHt) * sh);
      S.ring_slot_bytes = static_cast<int64_t>(S.ring_rows) * Wp * d.c * S.esize;
    }
  }

  // ---- MMA groups ---------------------------------------------------------
  int64_t gs = gs_req;
  if (gs == 0) {
    int64_t best = 0;
    for (int64_t g = 1; g <= r; ++g) {
      if (r % g || (g * d.cout) % 32 || g * d.cout > kMaxAccCols) continue;
      if (best == 0 || (best * d.cout < 64)) best = g;
      if (best * d.cout >= 64) break;
    }
    gs = best;
  }
  if (gs == 0 || r % gs || (gs * d.cout) % 32 || gs * d.cout > kMaxAccCols) {
    S.plan = fallback(WF_REASON_UNSUPPORTED_CHANNELS, f);
    *out = S;
    return WF_OK;
  }
  const int64_t G = r / gs;
  S.Ng = static_cast<int>(gs * d.cout);
  // Two A stages must fit in shared memory even with no B operand and the smallest
  // region layout (SWIZZLE_32B with one core-column offset, 16-bit inputs only);
  // otherwise the N-tiling below fails for every budget -- decided here, before the
  // K-step searches, which dominate planning time for wide folded pixels
  int64_t b_room = 0;  // B bytes one SM can hold beside two A stages (an upper bound)
  {
    const int64_t plain = Q * NR * Wbox * 16;
    const int64_t region_lb = (in_dtype == WF_TF32) ? plain : std::min<int64_t>(plain, (NR * Wbox * 32 + 1023) / 1024 * 1024);
    const int64_t fixed_lb = kCtrlBytes + kStagingBytes + kTileM * 16 + 128 + kMaxAccCols * 4 + 1024;
    b_room = kSmemLimit - fixed_lb - 2 * sh * region_lb;
    if (b_room < 0) {
      S.plan = fallback(WF_REASON_NOT_PROFITABLE, f);
      *out = S;
      return WF_OK;
    }
  }
  // 2-byte outputs: 64-column chunks (16 bf16 = 32 B per thread and row);
  // tf32 (fp32 outputs): 32-column chunks (8 fp32 = 32 B).
  S.CH = (in_dtype != WF_TF32 && S.Ng % 64 == 0) ? 64 : 32;
  if (S.prod == 4 && S.CH != 32) S.prod = 3;  // the gather kernel is built for 32-column epilogue chunks
  if (S.prod == 5 || S.prod == 6) S.CH = 32;  // 576 threads: the 64-column epilogue would spill at the register cap
  std::vector<int64_t> lo(G), hi(G);
  for (int64_t g = 0; g < G; ++g) {
    lo[g] = INT64_MAX;
    hi[g] = -1;
    for (int64_t j = g * gs; j < (g + 1) * gs; ++j) {
      const int64_t off = ((-c0) * f + j * sw - d.pad_w) * d.c;
      lo[g] = std::min(lo[g], off / E2);
      hi[g] = std::max(hi[g], (off + d.kw * d.c - 1) / E2);
    }
  }
  // A group's B operand holds at least one K-step per two (kh, core column) cells of its window
  // (kpair's best case), and an N-tile's B is at most min(the 128 KB budget, the room beside two
  // A stages) per SM. When one group exceeds that, or all of them need more than kMaxNTiles
  // tiles, the N-tiling below fails for every budget: give up before the cover search, which
  // is the planner's expensive part for wide windows
  {
    const int64_t pr = (pair_req == 1) ? 2 : 1;
    const int64_t cap = pr * std::min<int64_t>(128 * 1024, b_room);
    int64_t total = 0;
    bool fits = cap > 0;
    for (int64_t g = 0; g < G && fits; ++g) {
      const int64_t lb = (d.kh * (hi[g] - lo[g] + 1) + 1) / 2 * static_cast<int64_t>(S.Ng) * 32;
      fits = lb <= cap;
      total += lb;
    }
    // and an N-tile holds whole groups of at most max_tile_cols accumulator columns (as below)
    const int64_t mt_est = d.n * ceil_div(OH, OHt);
    const int64_t tile_cols = (mt_est * 2 <= 148 && G > 1) ? S.Ng : kMaxAccCols;
    const int64_t per_tile = tile_cols / S.Ng;
    if (!fits || total > kMaxNTiles * cap || per_tile < 1 || ceil_div(G, per_tile) > kMaxNTiles) {
      S.plan = fallback(WF_REASON_NOT_PROFITABLE, f);
      *out = S;
      return WF_OK;
    }
  }
  // ---- 32-byte K-steps ("units": core columns (c, c+1)) covering each group's window
  // Legacy cover: starts lo, lo+2, ... A start c with c % Q == Q-1 straddles two
  // folded pixels and needs the shifted A region (25% more TMA pieces). When
  // Q >= 2 the planner also tries covers that never straddle (overlapping K
  // columns are zeroed in B for all but the first covering unit) and keeps
  // them when the merged MMA cost is no higher: fewer A views per kh, wider
  // merged MMAs, no shift region.
  std::vector<std::vector<int64_t>> U(G);
  for (int64_t g = 0; g < G; ++g)
    for (int64_t c = lo[g]; c <= hi[g]; c += 2) U[g].push_back(c);
  const int64_t max_col = kwf * Q - 1;  // last core column of the KW'*f*C window row
  auto mma_cost = [](int64_t n) { return std::max<int64_t>(n / 2, 32 + n / 4); };
  // merged cost of groups [g0, g1) in slot order `order` with unit sets `us`
  auto merged_cost = [&](const std::vector<int>& order, const std::vector<std::vector<int64_t>>& us) {
    std::vector<int64_t> starts;
    for (const auto& v : us) starts.insert(starts.end(), v.begin(), v.end());
    std::sort(starts.begin(), starts.end());
    starts.erase(std::unique(starts.begin(), starts.end()), starts.end());
    int64_t cost = 0;
    for (int64_t st : starts) {
      int run = 0;
      for (size_t k = 0; k <= order.size(); ++k) {
        const bool has = k < order.size() &&
                         std::find(us[order[k]].begin(), us[order[k]].end(), st) != us[order[k]].end();
        if (has) {
          ++run;
        } else if (run) {
          cost += mma_cost(run * static_cast<int64_t>(gs * d.cout));
          run = 0;
        }
      }
    }
    return cost;
  };
  auto best_order_cost = [&](const std::vector<std::vector<int64_t>>& us) {
    std::vector<int> order(us.size());
    std::iota(order.begin(), order.end(), 0);
    int64_t best = merged_cost(order, us);
    while (std::next_permutation(order.begin(), order.end())) best = std::min(best, merged_cost(order, us));
    return best;
  };
  if (Q >= 2) {
    // minimal non-straddling covers of [l, h]: two choices per K-step, so a wide
    // group window (e.g. 7 folded outputs of 8 fp32 channels: 52 core columns)
    // has 2^26 of them -- enumerate at most kMaxCovers (the joint search below
    // looks at <= 4096 combinations anyway)
    constexpr size_t kMaxCovers = 64;
    std::function<void(int64_t, int64_t, std::vector<int64_t>&, std::vector<std::vector<int64_t>>&)> covers =
        [&](int64_t p, int64_t h, std::vector<int64_t>& cur, std::vector<std::vector<int64_t>>& outv) {
          if (outv.size() >= kMaxCovers) return;
          if (p > h) {
            outv.push_back(cur);
            return;
          }
          for (int64_t st : {p, p - 1}) {
            if (st < 0 || st + 1 > max_col || st % Q == Q - 1) continue;
            cur.push_back(st);
            covers(st + 2, h, cur, outv);
            cur.pop_back();
          }
        };
    // column tiles of at most 256 accumulator columns, searched jointly (<= 5 groups)
    for (int64_t g0 = 0; g0 < G;) {
      int64_t g1 = g0;
      while (g1 < G && (g1 - g0 + 1) * S.Ng <= kMaxAccCols) ++g1;
      const int64_t ng = g1 - g0;
      std::vector<std::vector<std::vector<int64_t>>> cand(ng);
      bool ok = ng <= 5;
      for (int64_t k = 0; k < ng && ok; ++k) {
        std::vector<int64_t> cur;
        covers(lo[g0 + k], hi[g0 + k], cur, cand[k]);
        ok = !cand[k].empty();
      }
      if (ok) {
        std::vector<std::vector<int64_t>> legacy(U.begin() + g0, U.begin() + g1);
        const int64_t legacy_cost = best_order_cost(legacy);
        std::vector<size_t> idx(ng, 0);
        std::vector<std::vector<int64_t>> best_us;
        int64_t best = INT64_MAX;
        for (int guard = 0; guard < 512; ++guard) {
          std::vector<std::vector<int64_t>> us(ng);
          for (int64_t k = 0; k < ng; ++k) us[k] = cand[k][idx[k]];
          const int64_t c = best_order_cost(us);
          if (c < best) { best = c; best_us = us; }
          int64_t k = 0;
          while (k < ng && ++idx[k] == cand[k].size()) idx[k++] = 0;
          if (k == ng) break;
        }
        // accept up to `slack` percent more MMA cost: dropping the shift region
        // saves TMA pieces and A-operand reads the MMA cost model does not see
        int64_t slack = 0;
        if (const char* env = std::getenv("WF_COVER_SLACK")) slack = std::atoll(env);
        if (best * 100 <= legacy_cost * (100 + slack))
          for (int64_t k = 0; k < ng; ++k) U[g0 + k] = best_us[k];
      }
      g0 = g1;
    }
  }
  auto n_units = [&](int64_t g) { return static_cast<int64_t>(U[g].size()); };
  // ---- cross-kh core-column pairing (kpair) ---------------------------------
  // Every (kh, core column c) a group's window touches is one 16-byte core
  // column of A; the legacy cover rounds each kh row's window out to 32-byte
  // K-steps. kpair instead pairs two single core columns that feed the same
  // accumulator run -- (kh, c) with (kh', c), or any two leftovers -- into one
  // K=16 MMA whose descriptor LBO is the distance between them. Chosen when the
  // measured-cycle cost model says it is cheaper (WF_KPAIR=0/1 forces it).
  const int64_t KHn = d.kh;
  auto kpair_mmas = [&](const std::vector<int>& ord) {  // ord: slot -> group
    return build_kpair(ord, lo, hi, static_cast<int>(KHn), S.Ng, max_col);
  };
  auto kpair_cost = [&](const std::vector<int>& ord) {
    int64_t c = 0;
    for (const PMma& m : kpair_mmas(ord)) c += mma_cost(static_cast<int64_t>(m.len) * S.Ng);
    return c;
  };
  auto best_kpair_order = [&](std::vector<int> ord, int64_t* cost) {
    std::vector<int> best_ord = ord;
    int64_t best = kpair_cost(ord);
    if (ord.size() <= 6) {
      std::sort(ord.begin(), ord.end());
      do {
        const int64_t c = kpair_cost(ord);
        if (c < best) { best = c; best_ord = ord; }
      } while (std::next_permutation(ord.begin(), ord.end()));
    }
    *cost = best;
    return best_ord;
  };
  {
    const char* env = std::getenv("WF_KPAIR");
    bool use = false;
    if (kpair_req >= 0) {
      use = kpair_req == 1;
    } else if (env && env[0] == '1') {
      use = true;
    } else if (!(env && env[0] == '0')) {
      int64_t legacy = 0, kp = 0;
      for (int64_t g0 = 0; g0 < G;) {  // column tiles of <= 256 accumulator columns, as above
        int64_t g1 = g0;
        while (g1 < G && (g1 - g0 + 1) * S.Ng <= kMaxAccCols) ++g1;
        std::vector<std::vector<int64_t>> us(U.begin() + g0, U.begin() + g1);
        legacy += KHn * best_order_cost(us);
        std::vector<int> ord(static_cast<size_t>(g1 - g0));
        std::iota(ord.begin(), ord.end(), static_cast<int>(g0));
        int64_t c = 0;
        best_kpair_order(ord, &c);
        kp += c;
        g0 = g1;
      }
      // a legacy cover that straddles folded pixels needs the shifted A region
      // (one more TMA box per residue, ~1/Q more pieces): charge it 10%
      bool straddle = false;
      for (int64_t g = 0; g < G; ++g)
        for (int64_t st : U[g]) straddle = straddle || (st % Q == Q - 1);
      use = kp * 10 < legacy * (straddle ? 11 : 10);
    }
    S.kpair = use;
  }
  S.need_shift = false;
  if (!S.kpair)
    for (int64_t g = 0; g < G; ++g)
      for (int64_t st : U[g])
        if (st % Q == Q - 1) S.need_shift = true;
  S.units = U;
  // A layout. Without straddling K-steps (and 2-byte inputs), every K-step is
  // 32 contiguous bytes inside one folded pixel: the A tile is kept as one
  // SWIZZLE_32B region per in-pixel offset q used ([row][folded col][32 B],
  // one 32-byte TMA piece per K-step; row-shifted views verified in
  // tools/probes/sw32_probe.cu). Otherwise the canonical no-swizzle layout of
  // 16-byte core columns ([q][row][folded col][16 B], + the shift region).
  S.sw32 = !S.kpair && !S.need_shift && Q >= 2 && in_dtype != WF_TF32;
  S.qs.clear();
  if (S.sw32) {
    for (int64_t g = 0; g < G; ++g)
      for (int64_t st : U[g])
        if (std::find(S.qs.begin(), S.qs.end(), static_cast<int>(st % Q)) == S.qs.end())
          S.qs.push_back(static_cast<int>(st % Q));
    std::sort(S.qs.begin(), S.qs.end());
    // the launch holds at most 4 region coordinates (ConvArgs::qcoord): wider
    // pixels (e.g. stride 3 -> f = 24, 9 core columns) keep the no-swizzle layout
    if (S.qs.size() > 4) {
      S.sw32 = false;
      S.qs.clear();
    }
  }
  if (S.sw32 && (S.prod == 4 || S.prod == 5 || S.prod == 6)) S.prod = 3;  // the gather warps / ring maps: no-swizzle layout only
  if (S.sw32) {
    S.lbo_a = 16;  // unused by SWIZZLE_32B K-major descriptors
    S.qregion_bytes = static_cast<int>((NR * Wbox * 32 + 1023) / 1024 * 1024);
    S.region_bytes = static_cast<int>(S.qs.size()) * S.qregion_bytes;
  } else {
    S.lbo_a = static_cast<int>(NR * Wbox * 16);
    S.region_bytes = static_cast<int>((((Q + (S.need_shift ? 1 : 0)) * S.lbo_a) + 127) / 128 * 128);
  }
  S.stage_bytes = static_cast<int>(sh) * S.region_bytes;
  S.tile_shift = static_cast<int>(OHt * Wbox * (S.sw32 ? 32 : 16));  // A bytes between the stage's tiles
  const int64_t block_bytes = static_cast<int64_t>(S.Ng) * 32;  // 2 core cols x Ng rows x 16 B
  auto group_b_bytes = [&](int64_t g) { return d.kh * n_units(g) * block_bytes; };
  // B bytes of the N-tile holding groups [g0, g1) (kpair: as built in slot order g0, g0+1, ...)
  auto tile_b_bytes = [&](int64_t g0, int64_t g1) {
    int64_t bytes = 0;
    if (S.kpair) {
      std::vector<int> ord(static_cast<size_t>(g1 - g0));
      std::iota(ord.begin(), ord.end(), static_cast<int>(g0));
      for (const PMma& m : kpair_mmas(ord)) bytes += static_cast<int64_t>(m.len) * S.Ng * 32;
    } else {
      for (int64_t g = g0; g < g1; ++g) bytes += group_b_bytes(g);
    }
    return bytes;
  };

  // ---- N-tiles and shared-memory budget ------------------------------------
  const int ctrl_bytes = kCtrlBytes;
  const int staging = kStagingBytes;   // 4 epilogue warps x 2 x 2 KB
  const int a_pad = kTileM * 16;
  const int bias_bytes = kMaxAccCols * 4;
    // raw input staging: the row producers' ring of row slots (prod 1/2), or
  // two slots holding a stage unit's contiguous row span (prod 4)
  const int64_t unit_rows = std::min<int64_t>(d.h, (tps * OHt - 1) * sh + d.kh);
  const int64_t unit_slot = (unit_rows * d.w * d.c * S.esize + 32 + 127) / 128 * 128;
  const int64_t ring = (S.prod == 1 || S.prod == 2) ? static_cast<int64_t>(kRawSlots) * raw_slot_bytes_for(d.w * d.c * S.esize)
                       : (S.prod == 4 ? 2 * unit_slot : 0);
  // A stages that fit beside a resident B of max_b bytes (>= 2, else false)
  auto fit_stages = [&](int64_t max_b) {
    const int64_t fixed = ctrl_bytes + staging + a_pad + 128 + (max_b + 127) / 128 * 128 + bias_bytes + ring + 1024;
    int stages = 0;
    for (int st2 = 4; st2 >= 2; --st2)
      if (fixed + static_cast<int64_t>(st2) * S.stage_bytes <= kSmemLimit) { stages = st2; break; }
    if (stages < 2) return false;
    S.stages = stages;
    S.b_smem_bytes = static_cast<int>((max_b + 127) / 128 * 128);
    S.smem_bytes = static_cast<int>(fixed + static_cast<int64_t>(stages) * S.stage_bytes);
    return true;
  };
  const int pr = (pair_req == 1) ? 2 : 1;  // CTA pairs: each SM holds half of every B block
  // Latency-bound launches (fewer M tiles than half the SMs, e.g. batch 1):
  // one group per N-tile multiplies the CTAs and shrinks the B each one loads.
  const int64_t mtiles_est = d.n * ceil_div(OH, OHt);
  const int64_t max_tile_cols = (mtiles_est * 2 <= 148 && G > 1) ? S.Ng : kMaxAccCols;
  int64_t b_budget = 128 * 1024 * pr;
  for (int attempt = 0; attempt < 8; ++attempt) {
    S.ntiles.clear();
    bool ok = true;
    int64_t g = 0;
    while (g < G) {
      NTile t{};
      t.g0 = static_cast<int>(g);
      int64_t cols = 0, bytes = 0;
      while (g < G && cols + S.Ng <= max_tile_cols && tile_b_bytes(t.g0, g + 1) <= b_budget) {
        cols += S.Ng;
        ++g;
        bytes = tile_b_bytes(t.g0, g);
      }
      if (g == t.g0) { ok = false; break; }
      t.g1 = static_cast<int>(g);
      t.col0 = static_cast<int>(t.g0 * S.Ng);
      t.cols = static_cast<int>(cols);
      t.b_bytes = bytes;
      S.ntiles.push_back(t);
    }
    if (!ok || S.ntiles.size() > static_cast<size_t>(kMaxNTiles)) {
      S.plan = fallback(WF_REASON_NOT_PROFITABLE, f);
      *out = S;
      return WF_OK;
    }
    int64_t max_b = 0;
    for (auto& t : S.ntiles) max_b = std::max(max_b, t.b_bytes);
    if (fit_stages((max_b + pr - 1) / pr)) break;
    b_budget /= 2;
    if (attempt == 7 || b_budget < block_bytes) {
      S.plan = fallback(WF_REASON_NOT_PROFITABLE, f);
      *out = S;
      return WF_OK;
    }
  }

  // ---- the schedule: per N-tile, kh -> unit -> run of groups -----------------
  // Groups that start a unit at the same core column u read the SAME A view;
  // when they sit in adjacent accumulator slots one MMA with N = Ng * run
  // serves them all (A is read from shared memory once). The slot order of
  // each N-tile is chosen to maximise such runs under a per-MMA cost model
  // measured on B200 (tools/probes/mma_probe.cu: N=64 -> 55, 128 -> 67,
  // 256 -> 128 cycles; shared-memory operand reads bound small N).
  auto unit_set = [&](int64_t g) { return U[g]; };
  // runs of one N-tile for a slot order: (u, first slot, number of slots)
  struct Run { int64_t u; int slot0, len; };
  auto runs_for = [&](const NTile& t, const std::vector<int>& order) {
    std::vector<int> slot_of(G, -1);
    for (size_t sidx = 0; sidx < order.size(); ++sidx) slot_of[order[sidx]] = static_cast<int>(sidx);
    std::vector<int64_t> us;
    for (int g = t.g0; g < t.g1; ++g)
      for (int64_t u : unit_set(g)) us.push_back(u);
    std::sort(us.begin(), us.end());
    us.erase(std::unique(us.begin(), us.end()), us.end());
    std::vector<Run> runs;
    for (int64_t u : us) {
      std::vector<int> slots;
      for (int g = t.g0; g < t.g1; ++g) {
        const auto uu = unit_set(g);
        if (std::find(uu.begin(), uu.end(), u) != uu.end()) slots.push_back(slot_of[g]);
      }
      std::sort(slots.begin(), slots.end());
      for (size_t i = 0; i < slots.size();) {
        size_t k = i + 1;
        while (k < slots.size() && slots[k] == slots[k - 1] + 1) ++k;
        runs.push_back({u, slots[i], static_cast<int>(k - i)});
        i = k;
      }
    }
    return runs;
  };
  auto order_cost = [&](const NTile& t, const std::vector<int>& order) {
    int64_t c = 0;
    for (const Run& rn : runs_for(t, order)) c += mma_cost(static_cast<int64_t>(rn.len) * S.Ng);
    return c;
  };
  S.entries.clear();
  S.entry_cc0.clear();
  S.entry_cc1.clear();
  S.entry_lbo.clear();
  S.order.assign(static_cast<size_t>(G), 0);
  // byte offset of core column c of kh's window row inside an A stage (no-swizzle layout)
  auto cc_addr = [&](int64_t kh, int64_t c) {
    const int64_t delta = kh - d.pad_h;
    const int b = static_cast<int>(pos_mod(delta, sh));
    const int a = static_cast<int>((delta - b) / sh);
    return static_cast<uint32_t>(b * S.region_bytes + ((a - S.amin[b]) * Wbox + c / Q) * 16 + (c % Q) * S.lbo_a);
  };
  auto cc_word = [](int64_t kh, int64_t c, uint32_t mask) {
    return static_cast<uint32_t>(kh) | (static_cast<uint32_t>(c) << 8) | (mask << 16);
  };
  int64_t b_cursor = 0;
  for (auto& t : S.ntiles) {
    std::vector<int> order;
    for (int g = t.g0; g < t.g1; ++g) order.push_back(g);
    t.entry0 = static_cast<int>(S.entries.size());
    t.b_off = b_cursor;
    uint32_t boff = 0;
    if (S.kpair) {
      int64_t cst = 0;
      order = best_kpair_order(order, &cst);
      for (size_t sidx = 0; sidx < order.size(); ++sidx) S.order[t.g0 + sidx] = order[sidx];
      const std::vector<PMma> mm = kpair_mmas(order);
      std::vector<std::pair<int, int>> rr;
      for (const PMma& m : mm) rr.push_back({m.slot0, m.len});
      std::vector<int> seq;
      if (!zero_init_order(rr, static_cast<int>(order.size()), &seq))
        return make_schedule_tps(d, f_req, gs_req, in_dtype, tps, out, err, 0, pair_req);
      std::vector<char> touched(order.size(), 0);
      for (int k : seq) {
        const PMma& m = mm[k];
        int i0 = 0, i1 = 1;  // core column 0 of the K-step = the lower shared-memory address
        if (cc_addr(m.kh[1], m.c[1]) < cc_addr(m.kh[0], m.c[0])) std::swap(i0, i1);
        const uint32_t a0 = cc_addr(m.kh[i0], m.c[i0]), a1 = cc_addr(m.kh[i1], m.c[i1]);
        MmaEntry e{};
        e.a_off = a0;
        e.b_off = boff;
        const int64_t n = static_cast<int64_t>(m.len) * S.Ng;
        boff += static_cast<uint32_t>(n * 32);
        const bool acc = touched[m.slot0] != 0;  // zero_init_order: all or none of the run touched
        for (int q = 0; q < m.len; ++q) touched[m.slot0 + q] = 1;
        e.meta = static_cast<uint32_t>(m.kh[i0]) | (static_cast<uint32_t>(m.c[i0]) << 8) |
                 (static_cast<uint32_t>(m.slot0) << 16) | (static_cast<uint32_t>(n >> 3) << 22) |
                 (acc ? 0x80000000u : 0u);
        e.tmem_col = static_cast<uint32_t>(m.slot0 * S.Ng);
        S.entries.push_back(e);
        S.entry_cc0.push_back(cc_word(m.kh[i0], m.c[i0], m.mask[i0]));
        S.entry_cc1.push_back(cc_word(m.kh[i1], m.c[i1], m.mask[i1]));
        S.entry_lbo.push_back(a1 - a0);
      }
      t.b_bytes = boff;
    } else {
      if (t.g1 - t.g0 <= 8) {  // exhaustive over slot orders (<= 40320)
        std::vector<int> cand = order;
        int64_t best = order_cost(t, order);
        while (std::next_permutation(cand.begin(), cand.end())) {
          const int64_t c = order_cost(t, cand);
          if (c < best) { best = c; order = cand; }
        }
      }
      for (size_t sidx = 0; sidx < order.size(); ++sidx) S.order[t.g0 + sidx] = order[sidx];
      const std::vector<Run> runs = runs_for(t, order);
      // zero-init: at kh == 0 every group's first MMA must not accumulate, so the
      // kh == 0 runs are ordered such that each one meets either only untouched
      // groups (accumulate = 0) or only touched ones (backtracking, few runs)
      std::vector<Run> first = runs;
      {
        std::vector<std::pair<int, int>> rr;
        for (const Run& rn : runs) rr.push_back({rn.slot0, rn.len});
        std::vector<int> seq;
        if (zero_init_order(rr, static_cast<int>(order.size()), &seq))
          for (size_t k = 0; k < seq.size(); ++k) first[k] = runs[seq[k]];
      }
      bool ok_init = true;
      for (int64_t kh = 0; kh < d.kh; ++kh) {
        const int64_t delta = kh - d.pad_h;
        const int b = static_cast<int>(pos_mod(delta, sh));
        const int a = static_cast<int>((delta - b) / sh);
        std::vector<char> touched(order.size(), 0);
        for (const Run& rn : (kh == 0 ? first : runs)) {
          const int64_t u = rn.u;  // first core column of the pair
          const int64_t kp = u / Q, q = u % Q;
          MmaEntry e{};
          if (S.sw32) {
            const int qi = static_cast<int>(std::find(S.qs.begin(), S.qs.end(), static_cast<int>(q)) - S.qs.begin());
            e.a_off = static_cast<uint32_t>(b * S.region_bytes + qi * S.qregion_bytes + ((a - S.amin[b]) * Wbox + kp) * 32);
          } else {
            e.a_off = static_cast<uint32_t>(b * S.region_bytes + ((a - S.amin[b]) * Wbox + kp) * 16 + q * S.lbo_a);
          }
          e.b_off = boff;
          const int64_t n = static_cast<int64_t>(rn.len) * S.Ng;
          boff += static_cast<uint32_t>(n * 32);
          bool acc = true;
          if (kh == 0) {
            int nt = 0;
            for (int k = 0; k < rn.len; ++k) nt += touched[rn.slot0 + k];
            if (nt != 0 && nt != rn.len) ok_init = false;
            acc = (nt != 0);
            for (int k = 0; k < rn.len; ++k) touched[rn.slot0 + k] = 1;
          }
          e.meta = static_cast<uint32_t>(kh) | (static_cast<uint32_t>(u) << 8) |
                   (static_cast<uint32_t>(rn.slot0) << 16) | (static_cast<uint32_t>(n >> 3) << 22) |
                   (acc ? 0x80000000u : 0u);
          e.tmem_col = static_cast<uint32_t>(rn.slot0 * S.Ng);
          S.entries.push_back(e);
          // core column u of a step is owned by the group's step at u - 1 if it has one
          uint32_t mask0 = 0;
          for (int k = 0; k < rn.len; ++k) {
            const auto& ug = U[order[rn.slot0 + k]];
            if (std::find(ug.begin(), ug.end(), u - 1) == ug.end()) mask0 |= 1u << k;
          }
          S.entry_cc0.push_back(cc_word(kh, u, mask0));
          S.entry_cc1.push_back(cc_word(kh, u + 1, (1u << rn.len) - 1u));
          S.entry_lbo.push_back(static_cast<uint32_t>(S.lbo_a));
        }
      }
      if (!ok_init) {  // cannot happen with disjoint per-group units; keep the planner total
        S.plan = fallback(WF_REASON_NOT_PROFITABLE, f);
        *out = S;
        return WF_OK;
      }
      if (static_cast<int64_t>(boff) != t.b_bytes) {
        *err = "internal: B operand bytes of a merged schedule differ from the plan";
        return WF_INVALID_ARGUMENT;
      }
    }
    t.entries = static_cast<int>(S.entries.size()) - t.entry0;
    // Half-split accumulator release: MMAs writing only the lower half of the
    // columns go first, so the next tile's lower-half MMAs can start as soon as
    // the epilogue has drained that half (1.5 accumulator buffers in effect).
    {
      const int mid = t.cols / 2;
      bool clean = (t.cols / S.CH) % 2 == 0 && mid % S.CH == 0;
      std::vector<int> lo_i, hi_i;
      for (int i = t.entry0; i < t.entry0 + t.entries && clean; ++i) {
        const MmaEntry& e = S.entries[i];
        const int c0e = static_cast<int>(e.tmem_col), ne = static_cast<int>((e.meta >> 22) & 0x1FFu) * 8;
        if (c0e + ne <= mid) lo_i.push_back(i);
        else if (c0e >= mid) hi_i.push_back(i);
        else clean = false;
      }
      if (clean && !lo_i.empty() && !hi_i.empty()) {
        std::vector<int> perm = lo_i;
        perm.insert(perm.end(), hi_i.begin(), hi_i.end());
        auto permute = [&](auto& v) {
          auto old = v;
          for (size_t k = 0; k < perm.size(); ++k) v[t.entry0 + k] = old[perm[k]];
        };
        permute(S.entries);
        permute(S.entry_cc0);
        permute(S.entry_cc1);
        permute(S.entry_lbo);
        t.split = static_cast<int>(lo_i.size());
      }
    }
    b_cursor += t.b_bytes;
  }
  if (S.kpair) {  // exact B sizes: the A stages must still fit beside the largest
    int64_t max_b = 0;
    for (const auto& t : S.ntiles) max_b = std::max(max_b, t.b_bytes);
    if (!fit_stages((max_b + pr - 1) / pr)) return make_schedule_tps(d, f_req, gs_req, in_dtype, tps, out, err, 0, pair_req);
  }

  // ---- plan facts -----------------------------------------------------------
  wf_fold_plan& p = S.plan;
  p = wf_fold_plan{};
  p.status = WF_FOLD_APPLY;
  p.reason = WF_REASON_NONE;
  p.f = f;
  p.r = r;
  p.c0 = c0;
  p.kw_f = kwf;
  p.k_f = d.kh * kwf * f * d.c;
  p.cout_f = r * d.cout;
  p.in_dtype = in_dtype;
  p.elem_bytes = S.esize;
  p.oh = OH;
  p.ow = OW;
  p.wf = Wf;
  p.wfo = Wfo;
  p.units_per_px = Q;
  p.group_size = gs;
  p.n_groups = G;
  p.n_tiles = static_cast<int64_t>(S.ntiles.size());
  p.tile_rows = OHt;
  p.wbox = Wbox;
  p.nrows = NR;
  if (S.entries.size() > static_cast<size_t>(kMaxEntries)) {  // e.g. 11x11 fp32 windows on wide pixels
    S.plan = fallback(WF_REASON_NOT_PROFITABLE, f);
    *out = S;
    return WF_OK;
  }
  p.mma_entries = static_cast<int64_t>(S.entries.size());
  // packed header: schedule table, the slot -> group order (int32 each), then
  // the (core column 0, core column 1) words of every entry
  p.table_bytes = (p.mma_entries * 24 + G * 4 + 127) / 128 * 128;
  p.packed_bytes = p.table_bytes + b_cursor;
  p.epi_chunk = S.CH;
  S.raw_slots = (S.prod == 4) ? 2 : (S.prod == 5 ? kRingSlots : (S.prod == 6 ? 0 : kRawSlots));
  S.raw_slot_bytes = (S.prod == 4) ? static_cast<int>(unit_slot)
                                   : ((S.prod == 5 || S.prod == 6) ? 0 : raw_slot_bytes_for(d.w * d.c * S.esize));
  p.variant = WF_VARIANT_FOLD;
  p.producer = S.prod;
  p.pitched_w = (S.prod == 3 || S.prod == 5) ? S.Wp : 0;
  p.workspace_bytes = (S.prod == 3) ? d.n * d.h * S.Wp * d.c * S.esize
                                    : (S.prod == 5 ? static_cast<int64_t>(kRingCtas) * kRingSlots * S.ring_slot_bytes : 0);
  S.ohb = ceil_div(OH, OHt);
  S.num_mtiles = d.n * S.ohb;
  // CTA pairs (cta_group::2, M = 256): each SM holds and reads half of every
  // B block. bf16/fp16 TMA plans with N a multiple of 16; more A stages fit.
  // Opt-in (pair_req 1): the pair MMA saves only ~10% at N=64 and nothing at
  // N>=128 (tools/probes/pair_probe.cu) while the pair synchronisation costs
  // more; halving B per SM did not pay for AlexNet either.
  {
    bool pair = pair_req == 1;
    pair = pair && in_dtype != WF_TF32 && (S.prod == 0 || S.prod == 3) && S.num_mtiles >= 2 && S.tps == 1;
    for (const MmaEntry& e : S.entries) pair = pair && (((e.meta >> 22) & 0x1FFu) * 8) % 16 == 0;
    if (pair_req == 1 && !pair) return make_schedule_tps(d, f_req, gs_req, in_dtype, tps, out, err, kpair_req, 0);
    if (pair) {
      int64_t max_b = 0;
      for (const auto& t : S.ntiles) max_b = std::max(max_b, t.b_bytes / 2);
      S.pair = 2;
      S.b_smem_bytes = static_cast<int>((max_b + 127) / 128 * 128);
      const int64_t fixed = kCtrlBytes + kTileM * 16 + 128 + S.b_smem_bytes + kMaxAccCols * 4 + 1024;
      for (int st2 = 6; st2 >= 2; --st2)
        if (fixed + static_cast<int64_t>(st2) * S.stage_bytes <= kSmemLimit) { S.stages = st2; break; }
    }
    p.cta_pair = S.pair;
    p.stage_tiles = S.tps;
    p.kstep_mode = S.kpair ? 1 : 0;
  }
  p.useful_macs = static_cast<uint64_t>(d.n) * OH * OW * d.cout * d.kh * d.kw * d.c;
  uint64_t issued_per_tile = 0;
  for (const MmaEntry& e : S.entries) issued_per_tile += static_cast<uint64_t>(kTileM) * ((e.meta >> 22) & 0x1FFu) * 8 * S.E;
  p.issued_macs = static_cast<uint64_t>(S.num_mtiles) * issued_per_tile;
  *out = std::move(S);
  return WF_OK;
}

}  // namespace

wf_status make_schedule_unfolded(const wf_conv_desc& d, wf_dtype in_dtype, Schedule* out, std::string* err) {
  wf_status st = validate_desc(d, err);
  if (st != WF_OK) return st;
  if (in_dtype != WF_BF16 && in_dtype != WF_F16) {
    *err = "the unfolded variant runs bf16/f16 inputs";
    return WF_INVALID_ARGUMENT;
  }
  Schedule S;
  S.esize = elem_bytes(in_dtype);
  S.E = 32 / S.esize;
  S.s = static_cast<int>(d.stride_h);
  S.ph = static_cast<int>(d.pad_h);
  S.pw = static_cast<int>(d.pad_w);
  S.prod = 2;
  const int64_t OH = (d.h + 2 * d.pad_h - d.kh) / d.stride_h + 1;
  const int64_t OW = (d.w + 2 * d.pad_w - d.kw) / d.stride_w + 1;
  if (d.cout % 32 != 0 || d.cout > kMaxAccCols) {
    S.plan = fallback(WF_REASON_UNSUPPORTED_CHANNELS, 1);
    *out = S;
    return WF_OK;
  }
  // M row = output pixel; per kh one window row of KW*C elements, U 32-byte
  // K-steps; every A view is materialised ([kh*U + u][core col][128 rows][16 B]).
  const int64_t U = ceil_div(d.kw * d.c * S.esize, 32);
  S.U = static_cast<int>(U);
  S.Q = 2;
  S.Ng = static_cast<int>(d.cout);
  S.CH = (S.Ng % 64 == 0) ? 64 : 32;
  S.lbo_a = kTileM * 16;
  S.region_bytes = 0;
  // kh rows per A stage: all of them when two stages fit, else split the
  // tile's K into ksplit sub-stages (AlexNet: 11 kh x 3 K-steps = 132 KB)
  const int64_t region = 2 * kTileM * 16;  // one (kh, K-step) view
  const int64_t b_total = d.kh * U * d.cout * 32;
  S.raw_slots = kRawSlots;
  S.raw_slot_bytes = raw_slot_bytes_for(d.w * d.c * S.esize);
  const int64_t fixed0 = kCtrlBytes + kTileM * 16 + 128 + (b_total + 127) / 128 * 128 + kMaxAccCols * 4 +
                         static_cast<int64_t>(S.raw_slots) * S.raw_slot_bytes + 1024;
  int64_t ksplit = 1;
  while (ksplit < 8 && fixed0 + 2 * ceil_div(d.kh, ksplit) * U * region > kSmemLimit) ++ksplit;
  const int64_t khs = ceil_div(d.kh, ksplit);
  ksplit = ceil_div(d.kh, khs);
  S.ksplit = static_cast<int>(ksplit);
  S.stage_bytes = static_cast<int>(khs * U * region);
  NTile t{};
  t.g0 = 0;
  t.g1 = 1;
  t.col0 = 0;
  t.cols = static_cast<int>(d.cout);
  t.b_bytes = d.kh * U * d.cout * 32;
  t.entry0 = 0;
  t.b_off = 0;
  S.order.assign(1, 0);
  uint32_t boff = 0;
  for (int64_t kh = 0; kh < d.kh; ++kh) {
    if (kh % khs == 0) {
      S.ks_kh0.push_back(static_cast<int>(kh));
      S.ks_entry0.push_back(static_cast<int>(S.entries.size()));
      S.ks_chunks.push_back(static_cast<int>(std::min(khs, d.kh - kh) * U * region / 16));
    }
    for (int64_t u = 0; u < U; ++u) {
      MmaEntry e{};
      e.a_off = static_cast<uint32_t>(((kh % khs) * U + u) * region);
      e.b_off = boff;
      boff += static_cast<uint32_t>(d.cout * 32);
      const bool acc = !(kh == 0 && u == 0);
      e.meta = static_cast<uint32_t>(kh) | (static_cast<uint32_t>(2 * u) << 8) |
               (static_cast<uint32_t>(d.cout >> 3) << 22) | (acc ? 0x80000000u : 0u);
      e.tmem_col = 0;
      S.entries.push_back(e);
      S.entry_cc0.push_back(static_cast<uint32_t>(kh) | (static_cast<uint32_t>(2 * u) << 8) | (1u << 16));
      S.entry_cc1.push_back(static_cast<uint32_t>(kh) | (static_cast<uint32_t>(2 * u + 1) << 8) | (1u << 16));
      S.entry_lbo.push_back(static_cast<uint32_t>(S.lbo_a));
    }
  }
  for (size_t k = 0; k < S.ks_entry0.size(); ++k)
    S.ks_entries.push_back(
        (k + 1 < S.ks_entry0.size() ? S.ks_entry0[k + 1] : static_cast<int>(S.entries.size())) - S.ks_entry0[k]);
  t.entries = static_cast<int>(S.entries.size());
  S.ntiles.push_back(t);
  const int64_t fixed = fixed0;
  S.stages = 0;
  for (int st2 = 4; st2 >= 2; --st2)
    if (fixed + static_cast<int64_t>(st2) * S.stage_bytes <= kSmemLimit) { S.stages = st2; break; }
  if (S.stages == 0 || S.entries.size() > static_cast<size_t>(kMaxEntries)) {
    S.plan = fallback(WF_REASON_NOT_PROFITABLE, 1);
    *out = S;
    return WF_OK;
  }
  S.b_smem_bytes = static_cast<int>((t.b_bytes + 127) / 128 * 128);
  wf_fold_plan& p = S.plan;
  p = wf_fold_plan{};
  p.status = WF_FOLD_APPLY;
  p.reason = WF_REASON_NONE;
  p.f = 1;
  p.r = 1;
  p.c0 = -d.pad_w;
  p.kw_f = d.kw;
  p.k_f = d.kh * d.kw * d.c;
  p.cout_f = d.cout;
  p.in_dtype = in_dtype;
  p.elem_bytes = S.esize;
  p.oh = OH;
  p.ow = OW;
  p.wf = d.w;
  p.wfo = OW;
  p.units_per_px = U;
  p.group_size = 1;
  p.n_groups = 1;
  p.n_tiles = 1;
  p.tile_rows = 0;
  p.wbox = 0;
  p.nrows = 0;
  p.mma_entries = static_cast<int64_t>(S.entries.size());
  p.table_bytes = (p.mma_entries * 24 + 4 + 127) / 128 * 128;
  p.packed_bytes = p.table_bytes + t.b_bytes;
  p.epi_chunk = S.CH;
  p.variant = WF_VARIANT_UNFOLDED;
  p.producer = 2;
  p.cta_pair = 1;
  p.stage_tiles = 1;
  const int64_t total = d.n * OH * OW;
  S.num_mtiles = ceil_div(total, kTileM);
  S.ohb = 1;
  p.useful_macs = static_cast<uint64_t>(total) * d.cout * d.kh * d.kw * d.c;
  p.issued_macs = static_cast<uint64_t>(S.num_mtiles) * S.entries.size() * kTileM * d.cout * S.E;
  *out = std::move(S);
  return WF_OK;
}

// Launch tuning knobs, decided once per plan (wf_fold_plan::launch_opts): the
// launch path never reads the environment. WF_NACC=2 two accumulator
// buffers, WF_EPI_PP=0/1 epilogue ping-pong off/on, WF_MCAST=1/0 force the
// multicast N-tile cluster on/off (default decided at launch preparation:
// conv_fold.cu; profiles/r2t_knobs_ab.log).
static int32_t launch_opts_from_env() {
  int32_t o = 0;
  if (const char* e = std::getenv("WF_NACC")) o |= (e[0] == '2') ? 1 : 0;
  if (const char* e = std::getenv("WF_EPI_PP")) o |= (e[0] == '1') ? (2 << 1) : (e[0] == '0' ? (1 << 1) : 0);
  if (const char* e = std::getenv("WF_MCAST")) o |= (e[0] == '0') ? 8 : (e[0] == '1' ? 16 : 0);
  return o;
}

wf_status make_schedule(const wf_conv_desc& d, int64_t f_req, int64_t gs_req, wf_dtype in_dtype, Schedule* out,
                        std::string* err, int kpair_req, int pair_req, int tps_req) {
  wf_status st = make_schedule_variant(d, f_req, gs_req, in_dtype, out, err, kpair_req, pair_req, tps_req);
  if (st == WF_OK && out->plan.status == WF_FOLD_APPLY) out->plan.launch_opts = launch_opts_from_env();
  return st;
}

wf_status schedule_from_plan(const wf_conv_desc& d, const wf_fold_plan& p,
                             Schedule* out, std::string* err) {
  if (p.status != WF_FOLD_APPLY) {
    *err = "plan is not an Apply plan";
    return WF_INVALID_ARGUMENT;
  }
  // the plan's own producer for unaligned rows, whatever WF_REPITCH / WF_GATHER say now
  ProdScope prod_scope(p.producer >= 3 ? p.producer : -1);
  wf_status st = (p.variant == WF_VARIANT_UNFOLDED)
                     ? make_schedule_unfolded(d, static_cast<wf_dtype>(p.in_dtype), out, err)
                     : make_schedule(d, p.f, p.group_size, static_cast<wf_dtype>(p.in_dtype), out, err,
                                     p.kstep_mode, p.cta_pair == 2 ? 1 : 0, p.stage_tiles);
  if (st != WF_OK) return st;
  if (out->plan.status != WF_FOLD_APPLY || out->plan.packed_bytes != p.packed_bytes ||
      out->plan.mma_entries != p.mma_entries) {
    *err = "plan does not match this conv descriptor";
    return WF_SHAPE_MISMATCH;
  }
  out->plan.launch_opts = p.launch_opts;
  if (out->prod != p.producer) {
    *err = "plan producer does not match this conv descriptor";
    return WF_SHAPE_MISMATCH;
  }
  return WF_OK;
}

}  // namespace wfb
