// conv_fold.cu -- host side of K2 (the folded conv): tensor maps, kernel
// arguments from the schedule, producer choice and launch. Device code:
// conv_kernel.cuh.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <utility>
#include <vector>

#include "conv_kernel.cuh"

namespace wfb {

// ============================== host side ==============================

namespace {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode(std::string* err) {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) *err = "cuTensorMapEncodeTiled unavailable (driver too old?)";
  return fn;
}

CUtensorMapDataType tmap_type(wf_dtype t) {
  switch (t) {
    case WF_BF16: return CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    case WF_F16: return CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    default: return CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  }
}

uint32_t pow2ceil(uint32_t v) {
  uint32_t p = 32;
  while (p < v) p <<= 1;
  return p;
}

}  // namespace

// Everything one launch needs, built once per (schedule, buffers, epilogue,
// device): kernel arguments with the MMA table, encoded tensor maps, the
// kernel, grid and shared memory. Immutable once built.
struct PreparedLaunch {
  // key
  const void *x, *workspace, *packed;
  const float* b_rep;
  void* y;
  wf_dtype out_dtype;
  uint32_t epilogue;
  int num_sms, device;
  // launch
  ConvArgs a;
  TmaMaps maps;
  const void* fn = nullptr;
  int grid = 0, block = 0, smem = 0, cluster = 1;
  bool pdl = true;  // programmatic dependent launch (WF_PDL=0 turns it off; read at prepare time)
  // operand epoch of this entry's last launch (~0: never launched): a launch
  // after a pack / bias write goes without PDL (note_operand_write)
  mutable std::atomic<uint64_t> epoch_seen{~0ull};
  // producer 3: re-pitch x into the workspace first
  bool repitch = false;
  long long rp_rows = 0;
  int rp_in = 0, rp_out = 0, rp_planes = 0;

  bool same(const void* x_, const void* ws_, const void* pk_, const float* b_, void* y_, wf_dtype o_, uint32_t e_,
            int sms_, int dev_) const {
    return x == x_ && workspace == ws_ && packed == pk_ && b_rep == b_ && y == y_ && out_dtype == o_ &&
           epilogue == e_ && num_sms == sms_ && device == dev_;
  }
};

namespace {

// Core-column planes in the re-pitch workspace (the TMA boxes then read whole
// folded-column runs of one core column instead of 16-byte pieces):
// no-swizzle single-CTA / multicast plans whose box run fits the 256-element
// box limit; WF_PLANES=0 turns it off. One definition for the conv launch and
// wf_repitch_input, so both agree on the layout.
bool repitch_planes(const Schedule& S, int es) {
  const char* ep = std::getenv("WF_PLANES");
  return !(ep && ep[0] == '0') && !S.sw32 && S.pair == 1 && S.plan.wbox * (16 / es) <= 256;
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is per (device context,
// function): remembered per device, under a lock.
cudaError_t ensure_smem(const void* fn, int device, int smem) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int, const void*>, int>> done;
  std::lock_guard<std::mutex> lk(mu);
  for (auto& e : done)
    if (e.first.first == device && e.first.second == fn) {
      if (e.second >= smem) return cudaSuccess;
      cudaError_t r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (r == cudaSuccess) e.second = smem;
      return r;
    }
  cudaError_t r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (r == cudaSuccess) done.push_back({{device, fn}, smem});
  return r;
}

wf_status prepare_conv(const Schedule& S, const wf_conv_desc& d, PreparedLaunch& L, std::string* err) {
  const void* x = L.x;
  const void* workspace = L.workspace;
  const void* packed = L.packed;
  const float* b_rep = L.b_rep;
  void* y = L.y;
  const wf_dtype out_dtype = L.out_dtype;
  const uint32_t epilogue = L.epilogue;
  const int num_sms = L.num_sms;
  ConvArgs& a = L.a;
  TmaMaps& maps = L.maps;
  const wf_fold_plan& p = S.plan;
  const wf_dtype in_t = static_cast<wf_dtype>(p.in_dtype);
  if (out_dtype != WF_F32 && out_dtype != WF_BF16 && out_dtype != WF_F16) {
    *err = "output dtype must be f32, bf16 or f16";
    return WF_INVALID_ARGUMENT;
  }
  if ((epilogue & WF_EPI_BIAS) && b_rep == nullptr) {
    *err = "bias epilogue requested without a replicated bias";
    return WF_INVALID_ARGUMENT;
  }
  if (((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(packed)) & 15u) ||
      (reinterpret_cast<uintptr_t>(y) & 31u)) {
    *err = "x and the packed filter must be 16-byte aligned, y 32-byte aligned";
    return WF_INVALID_ARGUMENT;
  }
  const int oes = elem_bytes(out_dtype);
  for (const auto& t : S.ntiles)
    if (t.cols % S.CH != 0) {
      *err = "N-tile width not a multiple of the epilogue chunk";
      return WF_UNSUPPORTED;
    }
  EncodeTiledFn encode = get_encode(err);
  if (!encode) return WF_CUDA_ERROR;

  static_assert(kMaxTable == kMaxEntries, "the planner's entry limit is the kernel's table size");
  if (S.entries.size() > static_cast<size_t>(kMaxTable)) {
    *err = "schedule too long for the constant bank";
    return WF_UNSUPPORTED;
  }
  std::memset(&a, 0, sizeof(a));
  std::memset(&maps, 0, sizeof(maps));
  a.bias = b_rep;
  a.out = static_cast<uint8_t*>(y);
  a.OHt = static_cast<int>(p.tile_rows);
  a.OH = static_cast<int>(p.oh);
  a.Wbox = static_cast<int>(p.wbox);
  a.Wfo = static_cast<int>(p.wfo);
  a.c0 = static_cast<int>(p.c0);
  a.s = S.s;
  a.ohb = static_cast<int>(S.ohb);
  a.num_mtiles = static_cast<int>(S.num_mtiles);
  a.res_mask = 0;
  for (int b = 0; b < S.s; ++b) {
    if (S.has_res[b]) a.res_mask |= 1u << b;
    a.amin[b] = S.amin[b];
  }
  const int Q = S.Q;
  // bytes each residue's boxes land per stage (the A full barrier's tx count)
  a.box_bytes = S.sw32 ? static_cast<int>(S.qs.size() * p.wbox * p.nrows * 32) : Q * S.lbo_a;
  a.shift_box_bytes = S.need_shift ? S.lbo_a : 0;
  a.shift_off = Q * S.lbo_a;
  a.region_bytes = S.region_bytes;
  a.stages = S.stages;
  a.stage_bytes = S.stage_bytes;
  a.n_tiles = static_cast<int>(S.ntiles.size());
  uint32_t max_cols = 0;
  const uint8_t* packed_b = static_cast<const uint8_t*>(packed) + p.table_bytes;
  for (int i = 0; i < a.n_tiles; ++i) {
    const NTile& t = S.ntiles[i];
    a.nt_entry0[i] = t.entry0;
    a.nt_entries[i] = t.entries;
    a.nt_split[i] = t.split;
    a.nt_col0[i] = t.col0;
    a.nt_cols[i] = t.cols;
    a.nt_bbytes[i] = static_cast<int>(t.b_bytes / S.pair);  // per CTA: half of every block in pair mode
    a.nt_bsrc[i] = reinterpret_cast<long long>(packed_b + t.b_off);
    max_cols = std::max<uint32_t>(max_cols, static_cast<uint32_t>(t.cols));
  }
  const uint32_t fmt = (in_t == WF_BF16) ? 1u : (in_t == WF_F16 ? 0u : 2u);
  const uint32_t idesc_base =
      (1u << 4) | (fmt << 7) | (fmt << 10) | ((static_cast<uint32_t>(kTileM * S.pair) >> 4) << 24);  // M = 128 / 256
  for (size_t i = 0; i < S.entries.size(); ++i) {
    const MmaEntry& e = S.entries[i];
    const uint32_t n8 = (e.meta >> 22) & 0x1FFu;  // N / 8 of this MMA
    const uint32_t lbo_b = n8 * 8u * 16u;         // B: [core col][N rows][16 B]
    const uint32_t lbo_a = S.entry_lbo.empty() ? static_cast<uint32_t>(S.lbo_a) : S.entry_lbo[i];
    a.table[i].x = (e.a_off >> 4) | ((lbo_a >> 4) << 16);
    a.table[i].y = ((e.b_off / S.pair) >> 4) | (((lbo_b / S.pair) >> 4) << 16);
    a.table[i].z = idesc_base | (n8 << 17) | (e.meta & 0x80000000u);
    a.table[i].w = e.tmem_col;
  }
  // absolute output column of every epilogue chunk (slot order -> groups)
  for (int i = 0; i < a.n_tiles; ++i) {
    const NTile& t = S.ntiles[i];
    for (int c = 0; c < t.cols / S.CH; ++c) {
      const int slot = (c * S.CH) / S.Ng;
      a.chunk_col[i][c] = S.order[t.g0 + slot] * S.Ng + (c * S.CH) % S.Ng;
    }
  }
  a.ctas_per_ntile = std::max(1, std::min<int>(num_sms / a.n_tiles, a.num_mtiles));
  if (S.pair == 2) a.ctas_per_ntile = std::max(2, a.ctas_per_ntile & ~1);  // whole CTA pairs
  a.tps = S.tps;
  a.uph = static_cast<int>((S.ohb + S.tps - 1) / S.tps);
  a.tile_shift = S.tile_shift;
  a.num_units = (S.tps > 1) ? static_cast<int>(d.n) * a.uph : static_cast<int>((a.num_mtiles + S.pair - 1) / S.pair);
  a.unit_stride = a.ctas_per_ntile / S.pair;
  if (S.tps > 1 && S.pair != 1) {
    *err = "two-tile stages run single-CTA";
    return WF_UNSUPPORTED;
  }
  a.row_bytes = p.cout_f * oes;
  a.acc_stride = pow2ceil(max_cols);
  // as many accumulator buffers as fit in the 512 TMEM columns (<= 4): the
  // MMAs run further ahead of the epilogue when an N-tile is narrow (MNv2 128)
  a.n_acc = (a.acc_stride <= 128 && !(p.launch_opts & 1)) ? 4 : 2;
  a.acc_shift = (a.n_acc == 4) ? 2 : 1;
  a.tmem_cols = a.n_acc * a.acc_stride;
  // epilogue ping-pong (the two warp groups alternate tiles): round 1 found it
  // +3% for a single narrow N-tile (MNv2, 128 columns) and -13% / -25% for R50 / VGG.
  // Round 2 (PDL, epilogue-staged bias): MNv2 0.205 -> 0.195 ms without it, so
  // it is opt-in (launch_opts bits 1-2 = 2, WF_EPI_PP=1 at plan time).
  a.epi_pp = 0;
  if (const int pp = (p.launch_opts >> 1) & 3) a.epi_pp = (pp == 2 && S.pair == 1) ? 1 : 0;
  a.epi_flags = static_cast<int>(epilogue);
  // Single-pass launches (every CTA gets at most one stage unit, e.g. batch 1):
  // extra A stages and accumulator buffers only cost shared memory and TMEM.
  // With one stage set (ksplit stages) and one accumulator per tile of the unit,
  // two CTAs fit on an SM, so under programmatic dependent launch the next
  // launch's CTAs become resident, initialise and load their B operand while
  // this launch still runs.
  if (a.num_units <= a.unit_stride && S.pair == 1 && !(p.launch_opts & 1)) {
    a.stages = std::max(1, std::min(a.stages, S.ksplit));  // (a.ksplit is filled in further down)
    while (a.n_acc > 1 && a.n_acc / 2 >= a.tps) {
      a.n_acc /= 2;
      --a.acc_shift;
    }
    a.tmem_cols = std::max(32u, static_cast<unsigned>(a.n_acc) * a.acc_stride);
  }
  // shared-memory carve-up (offsets from the 1024-aligned base)
  a.off_a = kCtrlBytes;
  a.off_b = a.off_a + a.stages * a.stage_bytes + kTileM * 16;
  a.off_b = (a.off_b + 127) / 128 * 128;
  a.off_bias = a.off_b + S.b_smem_bytes;
  // 0x4000 (profiling / cross-check): build the TMA-layout A tile with the row
  // producer instead -- same shared-memory image, so results are bit-identical
  const bool tf32 = (in_t == WF_TF32);
  const int prod =
      ((S.prod == 0 || S.prod >= 3) && (epilogue & WF_EPI_ROW_PRODUCER) && !tf32) ? 1
                                                                                                              : S.prod;
  a.prod = prod;
  a.off_raw = a.off_bias + kMaxAccCols * 4;
  // raw staging: the planner's slots for its own producer; the row-ring
  // cross-check (prod 1 forced on a TMA / gather plan) sizes its ring here
  a.raw_slots = (prod == S.prod) ? ((prod == 1 || prod == 2 || prod == 4 || prod == 5) ? S.raw_slots : 0) : kRawSlots;
  a.raw_slot_bytes = (prod == S.prod) ? S.raw_slot_bytes : raw_slot_bytes_for(d.w * d.c * S.esize);
  if (prod == 1 && S.prod != 1) {  // forced: make room for the ring by dropping A stages
    while (a.stages > 2 && a.off_raw + a.raw_slots * a.raw_slot_bytes + 1024 > kSmemLimit) {
      --a.stages;
      a.off_b = (a.off_a + a.stages * a.stage_bytes + kTileM * 16 + 127) / 128 * 128;
      a.off_bias = a.off_b + S.b_smem_bytes;
      a.off_raw = a.off_bias + kMaxAccCols * 4;
    }
  }
  const int smem = a.off_raw + a.raw_slots * a.raw_slot_bytes + 1024;
  a.rows_per_stage = 0;
  a.log_wbox = 0;
  while ((1 << a.log_wbox) < a.Wbox) ++a.log_wbox;
  for (int b = 0; b < S.s && (prod == 1 || prod == 4 || prod == 6); ++b) {  // folded raw rows of one stage (row producers)
    if (!S.has_res[b]) continue;
    const int rows = S.amax[b] - S.amin[b] + static_cast<int>(p.tile_rows) * S.tps;
    for (int i = 0; i < rows; ++i) {
      if (a.rows_per_stage >= kMaxStageRows) {
        *err = "too many raw rows per stage for the row producer";
        return WF_UNSUPPORTED;
      }
      a.row_b[a.rows_per_stage] = static_cast<signed char>(b);
      a.row_i[a.rows_per_stage] = static_cast<signed char>(i);
      a.row_a[a.rows_per_stage] = static_cast<signed char>(S.amin[b] + i);
      ++a.rows_per_stage;
    }
  }
  if (smem > kSmemLimit) {
    *err = "shared-memory budget exceeded";
    return WF_UNSUPPORTED;
  }

  // ---- software-gather producer arguments -------------------------------------
  const int es = S.esize;
  a.x = static_cast<const uint8_t*>(x);
  a.in_row_bytes = static_cast<long long>(d.w) * d.c * es;
  a.in_img_bytes = a.in_row_bytes * d.h;
  a.pix_bytes = (S.prod == 2 ? 1 : p.f) * d.c * es;
  a.H = static_cast<int>(d.h);
  a.Q = S.Q;
  a.Qr = S.Q + (S.need_shift ? 1 : 0);
  a.NR = static_cast<int>(p.nrows);
  a.lbo_a = S.lbo_a;
  a.OW = static_cast<int>(p.ow);
  a.r = static_cast<int>(p.r);
  a.Cout = static_cast<int>(d.cout);
  a.U = S.U;
  a.sw = static_cast<int>(d.stride_w);
  a.ph = static_cast<int>(d.pad_h);
  a.pw = static_cast<int>(d.pad_w);
  a.total_px = static_cast<long long>(d.n) * p.oh * p.ow;
  a.kh_count = static_cast<int>(d.kh);
  a.n_img = static_cast<int>(d.n);
  a.ksplit = S.ksplit;
  if (S.ksplit > kMaxKsplit) {
    *err = "too many A sub-stages";
    return WF_UNSUPPORTED;
  }
  for (int k = 0; k < S.ksplit && S.ksplit > 1; ++k) {
    a.ks_nkh[k] = (k + 1 < S.ksplit ? S.ks_kh0[k + 1] : static_cast<int>(d.kh)) - S.ks_kh0[k];
    a.ks_kh0[k] = S.ks_kh0[k];
    a.ks_entry0[k] = S.ks_entry0[k];
    a.ks_entries[k] = S.ks_entries[k];
  }

  // ---- producer 3: re-pitch x into the workspace (16-byte rows, Wp % f == 0) ------
  const void* xt = x;  // what the TMA boxes read
  if (prod == 3) {
    if (!workspace || (reinterpret_cast<uintptr_t>(workspace) & 15u)) {
      *err = "this plan needs a 16-byte aligned workspace of plan->workspace_bytes";
      return WF_INVALID_ARGUMENT;
    }
    L.repitch = true;
    L.rp_rows = d.n * d.h;
    L.rp_in = static_cast<int>(d.w * d.c * es);
    L.rp_out = static_cast<int>(S.Wp * d.c * es);
    if (repitch_planes(S, es)) {
      L.rp_planes = S.Q;
      a.planes_e2 = 16 / es;
    }
    xt = workspace;
  }
  // ---- producer 5: the gather warps re-pitch stage units into a ring of slots in the workspace
  if (prod == 5) {
    if (!workspace || (reinterpret_cast<uintptr_t>(workspace) & 15u)) {
      *err = "this plan needs a 16-byte aligned workspace of plan->workspace_bytes";
      return WF_INVALID_ARGUMENT;
    }
    a.ring = static_cast<uint8_t*>(const_cast<void*>(workspace));
    a.ring_rows = S.ring_rows;
    a.ring_rowpitch = static_cast<int>(S.Wp * d.c * es);
    a.amin_min = S.amin_min;
    a.ring_slot_bytes = S.ring_slot_bytes;
    xt = workspace;
  }
  // ---- A descriptor high word and the SWIZZLE_32B layout parameters -------------
  a.sw32 = S.sw32 ? 1 : 0;
  a.a_desc_hi = S.sw32 ? ((6u << 29) | (1u << 14) | (256u >> 4))   // SWIZZLE_32B, version 1, SBO 256 B
                       : ((1u << 14) | (128u >> 4));                // no swizzle, version 1, SBO 128 B
  a.nq = static_cast<int>(S.qs.size());
  a.qregion_bytes = S.qregion_bytes;
  for (int qi = 0; qi < a.nq && qi < 4; ++qi) {
    a.qcoord[qi] = S.qs[qi] * (16 / es);
    a.qbyte[qi] = S.qs[qi] * 16;
  }
  if (a.nq > 4) {
    *err = "too many SWIZZLE_32B regions";
    return WF_UNSUPPORTED;
  }
  // ---- input tensor maps (one 5-D view per H-stride residue) --------------------
  const cuuint64_t rowpitch = static_cast<cuuint64_t>((prod == 3 || prod == 5) ? S.Wp : d.w) * d.c * es;
  const cuuint64_t pix = static_cast<cuuint64_t>(p.f) * d.c * es;
  for (int b = 0; b < S.s && (prod == 0 || prod == 3 || prod == 5); ++b) {
    if (!S.has_res[b]) continue;
    // producer 5: the "image" dimension indexes ring slots of ring_rows rows each
    const cuuint64_t rows_b = static_cast<cuuint64_t>(((prod == 5 ? S.ring_rows : d.h) - b + S.s - 1) / S.s);
    if (S.sw32) {  // {pixel elements, folded col, input row of residue b, image}; 32-byte boxes
      cuuint64_t gdim4[4] = {static_cast<cuuint64_t>(p.f * d.c), static_cast<cuuint64_t>(p.wf), rows_b,
                             static_cast<cuuint64_t>(d.n)};
      cuuint64_t gstr4[3] = {pix, rowpitch * S.s, rowpitch * d.h};
      cuuint32_t box4[4] = {static_cast<cuuint32_t>(32 / es), static_cast<cuuint32_t>(p.wbox),
                            static_cast<cuuint32_t>(p.nrows), 1};
      cuuint32_t estr4[4] = {1, 1, 1, 1};
      void* gaddr4 = const_cast<uint8_t*>(static_cast<const uint8_t*>(xt) + b * rowpitch);
      const CUresult r4 = encode(&maps.in[b], tmap_type(in_t), 4, gaddr4, gdim4, gstr4, box4, estr4,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r4 != CUDA_SUCCESS) {
        *err = "cuTensorMapEncodeTiled(input, swizzle 32B) failed: " + std::to_string(static_cast<int>(r4));
        return WF_CUDA_ERROR;
      }
      continue;
    }
    if (prod == 3 && a.planes_e2) {  // {elements of a plane row, input row of residue b, plane, image}
      const cuuint64_t plane_bytes = static_cast<cuuint64_t>(p.wf) * 16;
      cuuint64_t gdim4[4] = {static_cast<cuuint64_t>(p.wf) * a.planes_e2, rows_b, static_cast<cuuint64_t>(Q),
                             static_cast<cuuint64_t>(d.n)};
      cuuint64_t gstr4[3] = {rowpitch * S.s, plane_bytes, rowpitch * d.h};
      cuuint32_t box4[4] = {static_cast<cuuint32_t>(p.wbox * a.planes_e2), static_cast<cuuint32_t>(p.nrows),
                            static_cast<cuuint32_t>(Q), 1};
      cuuint32_t estr4[4] = {1, 1, 1, 1};
      void* gaddr4 = const_cast<uint8_t*>(static_cast<const uint8_t*>(xt) + b * rowpitch);
      CUresult r4 = encode(&maps.in[b], tmap_type(in_t), 4, gaddr4, gdim4, gstr4, box4, estr4,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r4 == CUDA_SUCCESS && S.need_shift) {
        box4[2] = 1;  // plane 0 only, one folded column further
        r4 = encode(&maps.in_shift[b], tmap_type(in_t), 4, gaddr4, gdim4, gstr4, box4, estr4,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      }
      if (r4 != CUDA_SUCCESS) {
        *err = "cuTensorMapEncodeTiled(input, core-column planes) failed: " + std::to_string(static_cast<int>(r4));
        return WF_CUDA_ERROR;
      }
      continue;
    }
    cuuint64_t gdim[5] = {static_cast<cuuint64_t>(16 / es), static_cast<cuuint64_t>(p.wf), rows_b,
                          static_cast<cuuint64_t>(Q),
                          static_cast<cuuint64_t>(prod == 5 ? static_cast<int64_t>(kRingCtas) * S.raw_slots : d.n)};
    cuuint64_t gstr[4] = {pix, rowpitch * S.s, 16,
                          prod == 5 ? static_cast<cuuint64_t>(S.ring_slot_bytes) : rowpitch * d.h};
    cuuint32_t box[5] = {static_cast<cuuint32_t>(16 / es), static_cast<cuuint32_t>(p.wbox),
                         static_cast<cuuint32_t>(p.nrows), static_cast<cuuint32_t>(Q), 1};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    void* gaddr = const_cast<uint8_t*>(static_cast<const uint8_t*>(xt) + b * rowpitch);
    CUresult r = encode(&maps.in[b], tmap_type(in_t), 5, gaddr, gdim, gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS && S.need_shift) {
      box[3] = 1;  // core column 0 only
      r = encode(&maps.in_shift[b], tmap_type(in_t), 5, gaddr, gdim, gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) {
      *err = "cuTensorMapEncodeTiled(input) failed: " + std::to_string(static_cast<int>(r));
      return WF_CUDA_ERROR;
    }
  }

  const int grid = a.n_tiles * a.ctas_per_ntile;
  if (S.pair == 2 && (prod == 1 || prod == 2 || prod == 4 || prod == 6)) {
    *err = "the row producers run single-CTA plans";
    return WF_UNSUPPORTED;
  }
  if (prod == 5 && grid > kRingCtas) {
    *err = "more CTAs than the ring workspace was sized for";
    return WF_UNSUPPORTED;
  }
  if (tf32 && (S.CH != 32 || prod == 1 || prod == 2 || prod >= 4)) {
    *err = "tf32 plans use 32-column epilogue chunks and the TMA producer";
    return WF_UNSUPPORTED;
  }
  const int kind = tf32 ? 1 : 0;
  // two N-tiles as a 2-CTA cluster sharing each A stage by multicast
  // Default: on for TMA boxes of 16-byte pieces straight from x over >= 2 H-stride
  // residues (R50 f=16 "Cout=512": 3.86 -> 3.50 ms with it), off otherwise (VGG,
  // stride 1: 0.322 -> 0.298 ms without it; AlexNet's core-column-plane
  // workspace: 0.773 -> 0.766 ms without it). launch_opts bit 4 / bit 3 force on / off.
  const bool mc_default = (prod == 0 && S.s >= 2);
  const bool mc_on = (p.launch_opts & 16) ? true : ((p.launch_opts & 8) ? false : mc_default);
  const bool mc = mc_on && (prod == 0 || prod == 3 || prod == 5) && S.pair == 1 && !tf32 &&
                  a.n_tiles == 2 && a.ksplit == 1 && grid % 2 == 0;
  L.cluster = 1;
  if (mc) {
    L.fn = (prod == 5) ? conv_kernel_fn_mc5(out_dtype) : conv_kernel_fn_mc(out_dtype, S.CH);
    L.cluster = 2;
  } else if ((prod == 0 || prod == 3) && S.pair == 2) {
    L.fn = conv_kernel_fn_pair(out_dtype, S.CH);
    L.cluster = 2;
  } else if (prod == 0 || prod == 3) {
    L.fn = conv_kernel_fn<0>(kind, out_dtype, S.CH);
  } else if (prod == 1) {
    L.fn = conv_kernel_fn<1>(kind, out_dtype, S.CH);
  } else if (prod == 4 || prod == 6) {  // 6: the producer-4 kernel with a.prod == 6 (rows loaded from x)
    L.fn = conv_kernel_fn<4>(kind, out_dtype, S.CH);
  } else if (prod == 5) {
    L.fn = conv_kernel_fn<5>(kind, out_dtype, S.CH);
  } else {
    L.fn = conv_kernel_fn<2>(kind, out_dtype, S.CH);
  }
  if (!L.fn) {
    *err = "no conv kernel built for this producer / MMA kind / output type";
    return WF_UNSUPPORTED;
  }
  L.grid = grid;
  if (const char* e = std::getenv("WF_PDL")) L.pdl = e[0] != '0';
  L.block = (prod == 4 || prod == 6) ? 320 + 32 * kGatherWarps4
                        : (prod == 5 ? 320 + 32 * kGatherWarps5 : ((prod == 1 || prod == 2) ? 320 + 32 * kGatherWarps : 320));
  L.smem = smem;
  cudaError_t e = ensure_smem(L.fn, L.device, smem);
  if (e != cudaSuccess) {
    *err = std::string("cudaFuncSetAttribute(max dynamic shared memory) failed: ") + cudaGetErrorString(e);
    return WF_CUDA_ERROR;
  }
  return WF_OK;
}

std::atomic<uint64_t> g_operand_epoch{0};

cudaError_t launch_prepared(const PreparedLaunch& L, cudaStream_t st, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(L.grid);
  cfg.blockDim = dim3(L.block);
  cfg.dynamicSmemBytes = static_cast<size_t>(L.smem);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  unsigned n = 0;
  if (L.cluster > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = L.cluster;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  if (pdl) {  // the kernel's prologue (+ B load) overlaps the previous grid (griddepcontrol.wait guards the rest)
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = n ? attr : nullptr;
  cfg.numAttrs = n;
  void* args[2] = {const_cast<ConvArgs*>(&L.a), const_cast<TmaMaps*>(&L.maps)};
  return cudaLaunchKernelExC(&cfg, L.fn, args);
}

}  // namespace

wf_status launch_conv(const Schedule& S, const wf_conv_desc& d, const void* x, const void* workspace, const void* packed,
                      const float* b_rep, void* y, wf_dtype out_dtype, uint32_t epilogue, cudaStream_t st,
                      int num_sms, LaunchCache* cache, std::string* err) {
  int device = 0;
  if (cudaGetDevice(&device) != cudaSuccess) {
    *err = "cudaGetDevice failed";
    return WF_CUDA_ERROR;
  }
  if (num_sms <= 0) num_sms = sm_count(device);
  std::shared_ptr<const PreparedLaunch> L;
  if (cache) {
    std::lock_guard<std::mutex> lk(cache->mu);
    for (size_t i = 0; i < cache->entries.size(); ++i)
      if (cache->entries[i]->same(x, workspace, packed, b_rep, y, out_dtype, epilogue, num_sms, device)) {
        L = cache->entries[i];
        if (i) std::swap(cache->entries[i], cache->entries[0]);  // most recent first
        break;
      }
  }
  if (!L) {
    auto n = std::make_shared<PreparedLaunch>();
    n->x = x; n->workspace = workspace; n->packed = packed; n->b_rep = b_rep; n->y = y;
    n->out_dtype = out_dtype; n->epilogue = epilogue; n->num_sms = num_sms; n->device = device;
    wf_status ps = prepare_conv(S, d, *n, err);
    if (ps != WF_OK) return ps;
    L = n;
    if (cache) {
      std::lock_guard<std::mutex> lk(cache->mu);
      cache->entries.insert(cache->entries.begin(), n);
      if (cache->entries.size() > LaunchCache::kMax) cache->entries.pop_back();
    }
  }
  if (L->repitch && !(epilogue & WF_EPI_PREPITCHED)) {
    wf_status rs =
        launch_repitch(x, const_cast<void*>(workspace), L->rp_rows, L->rp_in, L->rp_out, L->rp_planes, st, err);
    if (rs != WF_OK) return rs;
  }
  const uint64_t ep = g_operand_epoch.load(std::memory_order_acquire);
  const bool pdl = L->pdl && L->epoch_seen.exchange(ep, std::memory_order_acq_rel) == ep;
  const cudaError_t e = launch_prepared(*L, st, pdl);
  if (e != cudaSuccess) {
    *err = std::string("conv_fold_kernel launch failed: ") + cudaGetErrorString(e);
    return WF_CUDA_ERROR;
  }
  return WF_OK;
}

wf_status launch_repitch_input(const Schedule& S, const wf_conv_desc& d, const void* x, void* workspace,
                               cudaStream_t st, std::string* err) {
  if (S.prod != 3) return WF_OK;
  if (!workspace || (reinterpret_cast<uintptr_t>(workspace) & 15u) || (reinterpret_cast<uintptr_t>(x) & 15u)) {
    *err = "x and the workspace must be 16-byte aligned";
    return WF_INVALID_ARGUMENT;
  }
  const int es = S.esize;
  return launch_repitch(x, workspace, d.n * d.h, static_cast<int>(d.w * d.c * es), static_cast<int>(S.Wp * d.c * es),
                        repitch_planes(S, es) ? S.Q : 0, st, err);
}

void note_operand_write() { g_operand_epoch.fetch_add(1, std::memory_order_acq_rel); }
uint64_t operand_epoch() { return g_operand_epoch.load(std::memory_order_acquire); }

int sm_count(int device) {
  static std::mutex mu;
  static std::vector<std::pair<int, int>> known;
  std::lock_guard<std::mutex> lk(mu);
  for (auto& k : known)
    if (k.first == device) return k.second;
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  known.push_back({device, n});
  return n;
}

}  // namespace wfb
