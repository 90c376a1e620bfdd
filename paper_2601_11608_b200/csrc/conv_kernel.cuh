// conv_kernel.cuh -- K2: the folded implicit-GEMM first-layer convolution
// kernel for sm_100a (device code; instantiated per producer in
// conv_prod{0,1,2}.cu, launched from conv_fold.cu).
//
// Replaces the reference hot loop widthfold::conv2d (src/refconv.cpp:57-78)
// run on the width-folded view (src/fold.cpp:113-143, a reshape) followed by
// bias_add (src/refconv.cpp:82-95) and reconstruct_output (src/fold.cpp:228-259,
// a reshape). One persistent, warp-specialised CTA per SM:
//
//   warp 0       producer. kProd 0: TMA -- per 128-row M tile one 5-D box per
//                H-stride residue lands the canonical K-major core-matrix
//                layout directly (plan.hpp explains the view), OOB = padding.
//                kProd 1/2: one bulk copy per raw input row into a slot
//                ring; transposer warps 10..11 build the A tile from it (16-byte
//                loads, any row alignment) builds the same folded layout
//                (AlexNet's 1362-byte pitch) or an explicit im2col layout
//                (the unfolded Cin=3 variant). Also bulk-copies the packed B.
//   warp 1       TMEM allocator + single-thread tcgen05.mma issuer, driven by
//                the schedule table built by plan.cpp; fp32 accumulators
//                double-buffered in TMEM.
//   warps 2..9   epilogue: tcgen05.ld.16x256b -> +bias -> ReLU -> convert ->
//                full-line 32-byte stores of final NHWC.
//
// Work split: CTA c serves N-tile (c % n_tiles) and M tiles
// local, local + ctas_per_ntile, ... -- the B operand of its N-tile stays
// resident in shared memory for the whole launch.
#pragma once

#include <cstdio>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "kernels.hpp"
#include "ptx.cuh"

namespace wfb {

constexpr int kMaxTable = 384;  // schedule entries per launch (constant bank)
#ifndef WFB_ISSUE_GROUP
#define WFB_ISSUE_GROUP 7
#endif
constexpr int kIssueGroup = WFB_ISSUE_GROUP;  // MMAs whose table words are loaded together
constexpr int kGatherWarps = 4;  // row-staged producer: transposer warps 10..13
// direct gather producer (kProd 4): warps 10..17 (row loads are latency-bound:
// more warps beat the 128-register cap of 16 warps)
constexpr int kGatherWarps4 = 8;
// L2-ring producer (kProd 5): warps 10..17 re-pitch each stage unit's input rows
// into a ring slot in global memory; warp 0 then loads the A stage from it by TMA
constexpr int kGatherWarps5 = 8;
constexpr int kMaxKsplit = 8;    // A stages per M tile (im2col kh ranges)
constexpr int kMaxStageRows = 64;  // folded raw rows per A stage (row producer)

struct ConvArgs {
  const float* bias;  // replicated bias (r*Cout fp32) or nullptr
  uint8_t* out;       // y (n, oh, ow, cout) NHWC
  int num_mtiles, ohb, OHt, OH, Wbox, Wfo, c0;
  int s;
  unsigned res_mask;
  int amin[kMaxResidues];
  int box_bytes, shift_box_bytes, region_bytes, shift_off;
  int stages, stage_bytes;
  int n_tiles, ctas_per_ntile;
  int nt_entry0[kMaxNTiles], nt_entries[kMaxNTiles], nt_col0[kMaxNTiles], nt_cols[kMaxNTiles];
  int nt_split[kMaxNTiles];       // lower-half MMAs of the N-tile (-1: no accumulator half-split)
  int num_units, unit_stride;     // M-tile units (pairs of M tiles in cta_group::2 mode) and the CTA stride
  unsigned a_desc_hi;             // A descriptor bits 32..63: SBO, version, layout (no swizzle / SWIZZLE_32B)
  int tps, uph, tile_shift;       // M tiles per A stage, stage units per image (tps > 1), A bytes between tiles
  int sw32, nq, qregion_bytes;    // SWIZZLE_32B A: one 32-byte-piece box per in-pixel offset
  int planes_e2;                  // > 0: the workspace holds core-column planes [q][folded col][16 B]
                                  // (re-pitch pass), 4-D boxes with whole-run inner pieces; value =
                                  // elements per 16-byte core column
  int qcoord[4];                  // sw32: element coordinate (in the pixel) of each region's box
  int qbyte[4];                   // sw32: the same offset in bytes
  int nt_bbytes[kMaxNTiles];
  long long nt_bsrc[kMaxNTiles];  // device address of the N-tile's packed B
  long long row_bytes;            // bytes of one folded output row = r*Cout*out_elem
  int chunk_col[kMaxNTiles][kMaxAccCols / 32];  // output column of each epilogue chunk
  unsigned acc_stride, tmem_cols;
  int n_acc, acc_shift;           // accumulator buffers in TMEM (2 or 4) and log2 of it
  int epi_pp;                     // epilogue ping-pong: warp groups alternate tiles
  int epi_flags;
  int off_a, off_b, off_bias;
  // software-gather producer (kProd 1: folded layout, 2: explicit im2col)
  const uint8_t* x;               // input base (16-byte aligned)
  long long in_row_bytes;         // W*C*elem (any alignment: AlexNet 1362 B)
  long long in_img_bytes;         // H*W*C*elem
  long long pix_bytes;            // folded pixel f*C*elem
  int H, Q, Qr, NR;               // core cols per pixel, regions per residue (+shift), rows per region
  int lbo_a;                      // bytes between core-column regions
  int prod;                       // A producer (plan.hpp Schedule::prod)
  int off_raw, raw_slots, raw_slot_bytes;  // staged-row ring (kProd 1/2) / the two raw unit slots (kProd 4)
                                           // / the L2 ring's slots per CTA (kProd 5, no shared memory)
  uint8_t* ring;                  // kProd 5: this launch's ring (workspace), ring_slots slots per CTA
  int ring_rows, ring_rowpitch;   // kProd 5: input rows per slot, re-pitched row bytes (16-byte multiple)
  int amin_min;                   // kProd 5: slot row 0 = input row (oh0 + amin_min) * s
  long long ring_slot_bytes;
  int rows_per_stage;             // folded: raw rows per A stage
  int log_wbox;                   // log2(Wbox)
  signed char row_b[kMaxStageRows], row_i[kMaxStageRows], row_a[kMaxStageRows];  // folded stage rows
  int kh_count, n_img;            // KH, N
  int ks_nkh[kMaxKsplit];         // im2col: kh rows per sub-stage
  // A stages per M tile (im2col: kh ranges; folded: 1) and their MMA / chunk ranges
  int ksplit;
  int ks_kh0[kMaxKsplit], ks_entry0[kMaxKsplit], ks_entries[kMaxKsplit], ks_chunks[kMaxKsplit];
  // output addressing: y(n, oh, ow, cout); folded column w' covers ow = w'*r + j
  int OW, r, Cout;
  // im2col producer / epilogue
  int U, sw, ph, pw;              // 32-byte K-steps per kh, W stride, padding
  long long total_px;             // N*OH*OW
  // schedule: x = (a_off>>4) | (lbo_a>>4)<<16, y = (b_off>>4) | (lbo_b>>4)<<16,
  // z = accumulate flag (bit 31), w = accumulator column
  uint4 table[kMaxTable];
};

struct TmaMaps {
  CUtensorMap in[kMaxResidues];
  CUtensorMap in_shift[kMaxResidues];  // core column 0 one folded column further (region Q)
};

// Profiling / diagnosis switches (the 0xFFFF00 bits of epi_flags; DESIGN.md
// 5.1b): compiled in only by a WFB_PROFILE=1 build (`make PROFILE=1`). A
// release build folds every check to false and the C-ABI rejects the bits.
#ifndef WFB_PROFILE
#define WFB_PROFILE 0
#endif
__device__ __forceinline__ bool prof(const ConvArgs& a, int bit) {
#if WFB_PROFILE
  return (a.epi_flags & bit) != 0;
#else
  (void)a;
  (void)bit;
  return false;
#endif
}

// Launch timeline of CTA 0 (PROFILE builds, TMA producer, switch 0x8000): %globaltimer
// stamps of each role's milestones in the control area, printed at exit.
__device__ __forceinline__ void tl_mark(const ConvArgs& a, uint8_t* gbase, int slot) {
#if WFB_PROFILE
  if ((a.epi_flags & 0x8000) && blockIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    reinterpret_cast<unsigned long long*>(gbase + 1536)[slot] = t;
  }
#else
  (void)a;
  (void)gbase;
  (void)slot;
#endif
}

template <typename OutT>
__device__ __forceinline__ uint32_t pack2(float lo, float hi);
template <>
__device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
template <>
__device__ __forceinline__ uint32_t pack2<__half>(float lo, float hi) {
  __half2 v = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// tcgen05.ld.16x256b with NREG/4 repetitions: 16 TMEM lanes x (NREG/2) columns.
template <int NREG>
__device__ __forceinline__ void tmem_ld_16x256b(uint32_t taddr, uint32_t (&r)[NREG], bool skip = false) {
  if (skip) {
#pragma unroll
    for (int k = 0; k < NREG; ++k) r[k] = taddr + k;  // profiling: no TMEM traffic
    return;
  }
  if constexpr (NREG == 32) ptx::tmem_ld_16x256b_x8(taddr, r); else ptx::tmem_ld_16x256b_x4(taddr, r);
}

// VPT consecutive output channels of one row -> global, 32-byte stores
// (kStream: L1::no_allocate + L2::evict_first).
template <typename OutT, int VPT, bool kStream>
__device__ __forceinline__ void store_row(uint8_t* dst, const float (&v)[VPT]) {
  auto st8 = [](uint8_t* p, const uint32_t* w) {
    if constexpr (kStream) ptx::st_global_v8_stream(p, w); else ptx::st_global_v8(p, w);
  };
  if constexpr (sizeof(OutT) == 4) {
    static_assert(VPT % 8 == 0, "fp32 rows are stored 8 values at a time");
#pragma unroll
    for (int q = 0; q < VPT / 8; ++q) {
      uint32_t pk[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) pk[k] = __float_as_uint(v[8 * q + k]);
      st8(dst + 32 * q, pk);
    }
  } else if constexpr (VPT == 16) {
    uint32_t pk[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) pk[k] = pack2<OutT>(v[2 * k], v[2 * k + 1]);
    st8(dst, pk);
  } else {
    static_assert(VPT == 8, "2-byte rows are 8 or 16 values");
    const uint4 w = make_uint4(pack2<OutT>(v[0], v[1]), pack2<OutT>(v[2], v[3]), pack2<OutT>(v[4], v[5]),
                               pack2<OutT>(v[6], v[7]));
    if constexpr (kStream) ptx::st_global_v4_stream(dst, w); else ptx::st_global_v4(dst, w);
  }
}

// ---- row-staged producer (kProd 1 / 2) -----------------------------------------
// The loader (warp 0, one lane) bulk-copies every raw input row a stage needs
// -- the 16-byte aligned superset [floor16(row), ceil16(row end)) -- into a
// ring of shared-memory slots; the transposer warps (10..11) turn each staged
// row into the stage's A layout with 16-byte shared-memory moves (funnel
// shifts when the row is not 16-byte aligned, e.g. AlexNet's 1362-byte rows)
// and zero-fill padding. Global memory is read once per row with one large
// copy instead of 16-byte TMA box pieces.

// Scalars of the row producer, read from the kernel parameters ONCE into
// registers: the shared-memory asm statements clobber "memory", so fields
// read through `a` inside the loops would be re-fetched from the constant
// bank every row (and the parameter block, with the MMA table, is larger
// than the constant cache).
struct RowProd {
  const uint8_t* x;
  long long in_img_bytes, total_px;
  int rb, pix, prod, Wbox, lw, Q, Qr, c0, lbo, region_bytes, s, H, n_img, ohb, OHt, OH, OW, U, sw, pw, ph;
  int rows_per_stage, ksplit, kh_count, raw_slots, raw_slot_bytes;
  int sw32, qregion_bytes;  // SWIZZLE_32B A layout (plan.hpp Schedule::sw32)
  uint32_t row_tab;  // shared address of the folded stage-row table: b | i << 8 | a << 16
};

// Launders a parameter value through a register: without it the compiler
// re-reads the field from the constant bank at every use (cheap to encode,
// but ~20+ cycles of latency on the transposers' serial per-row path).
__device__ __forceinline__ int opq(int v) {
  int r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}
__device__ __forceinline__ long long opq64(long long v) {
  long long r;
  asm volatile("mov.b64 %0, %1;" : "=l"(r) : "l"(v));
  return r;
}

__device__ __forceinline__ RowProd row_prod(const ConvArgs& a, uint32_t row_tab) {
  RowProd p;
  p.x = reinterpret_cast<const uint8_t*>(opq64(reinterpret_cast<long long>(a.x)));
  p.in_img_bytes = opq64(a.in_img_bytes);
  p.total_px = opq64(a.total_px);
  p.rb = opq(static_cast<int>(a.in_row_bytes));
  p.pix = opq(static_cast<int>(a.pix_bytes));
  p.prod = a.prod;
  p.Wbox = opq(a.Wbox);
  p.lw = opq(a.log_wbox);
  p.Q = opq(a.Q);
  p.Qr = opq(a.Qr);
  p.c0 = opq(a.c0);
  p.lbo = opq(a.lbo_a);
  p.region_bytes = opq(a.region_bytes);
  p.s = opq(a.s);
  p.H = opq(a.H);
  p.n_img = opq(a.n_img);
  p.ohb = opq(a.ohb);
  p.OHt = opq(a.OHt);
  p.OH = opq(a.OH);
  p.OW = opq(a.OW);
  p.U = opq(a.U);
  p.sw = opq(a.sw);
  p.pw = opq(a.pw);
  p.ph = opq(a.ph);
  p.rows_per_stage = opq(a.rows_per_stage);
  p.ksplit = opq(a.ksplit);
  p.kh_count = opq(a.kh_count);
  p.raw_slots = a.raw_slots;
  p.raw_slot_bytes = opq(a.raw_slot_bytes);
  p.sw32 = opq(a.sw32);
  p.qregion_bytes = opq(a.qregion_bytes);
  p.row_tab = row_tab;
  return p;
}

// Image and first output row of M tile k of stage unit u (this CTA's tile in pair mode).
template <int kPair>
__device__ __forceinline__ void tile_origin(const ConvArgs& a, int u, int k, uint32_t rank, int& n, int& oh0) {
  if (a.tps > 1) {
    n = u / a.uph;
    oh0 = ((u - n * a.uph) * a.tps + k) * a.OHt;
  } else {
    const int mt = u * kPair + static_cast<int>(rank);
    n = mt / a.ohb;
    oh0 = (mt - n * a.ohb) * a.OHt;
  }
}

// Raw rows of one A stage, enumerated identically by the loader and the
// transposers. Folded: row r = (residue b, region row i), input row
// (oh0 + a) * s + b with a = amin[b] + i. im2col: row r = (output row t of the
// tile, kh of the sub-stage), r = t * nkh + (kh - kh0).
struct StageRows {
  int count;       // rows in the stage
  int n0, oh0;     // folded: image and first output row of the tile
  long long g0;    // im2col: first global output row (n*OH + oh) of the tile
  int kh0, nkh;    // im2col: kh range of the sub-stage
};

template <int kProd>
__device__ __forceinline__ StageRows stage_rows(const ConvArgs& a, const RowProd& p, int mt, int ks) {
  StageRows sr;
  if constexpr (kProd == 1) {  // `mt` is the stage unit here (tps M tiles from tile_origin)
    tile_origin<1>(a, mt, 0, 0u, sr.n0, sr.oh0);
    sr.count = p.rows_per_stage;
    sr.g0 = 0;
    sr.kh0 = 0;
    sr.nkh = 0;
  } else {
    sr.kh0 = (p.ksplit == 1) ? 0 : a.ks_kh0[ks];
    sr.nkh = (p.ksplit == 1) ? p.kh_count : a.ks_nkh[ks];
    const long long P0 = static_cast<long long>(mt) * 128;
    const long long P1 = min(P0 + 127, p.total_px - 1);
    sr.g0 = P0 / p.OW;
    sr.count = static_cast<int>(P1 / p.OW - sr.g0 + 1) * sr.nkh;
    sr.n0 = 0;
    sr.oh0 = 0;
  }
  return sr;
}

// (image, input row) of stage row r; valid = inside the image (else zero-filled)
template <int kProd>
__device__ __forceinline__ bool stage_row(const RowProd& p, const StageRows& sr, int r, int& n, int& ih) {
  if constexpr (kProd == 1) {
    const uint32_t e = ptx::ld_shared_u32(p.row_tab + 4 * r);
    n = sr.n0;
    ih = (sr.oh0 + static_cast<int>(static_cast<int8_t>(e >> 16))) * p.s + static_cast<int>(e & 0xFF);
  } else {
    const int t = r / sr.nkh;
    const long long g = sr.g0 + t;
    n = static_cast<int>(g / p.OH);
    const int oh = static_cast<int>(g - static_cast<long long>(n) * p.OH);
    ih = oh * p.s - p.ph + sr.kh0 + (r - t * sr.nkh);
  }
  return ih >= 0 && ih < p.H && n < p.n_img;
}

// 16 bytes at row offset o of a staged row (slot holds the row from byte sh),
// bytes outside [0, rb) read as zero.
__device__ __forceinline__ uint4 raw16(uint32_t slot, int sh, int o, int rb) {
  const uint4 z = make_uint4(0u, 0u, 0u, 0u);
  if (o >= rb || o + 16 <= 0) return z;
  const int ad = sh + o;
  const int a0 = ad & ~15;
  const int s2 = ad - a0;
  uint32_t w0 = 0, w1 = 0, w2 = 0, w3 = 0;
  if (a0 >= 0) {
    const uint4 v0 = ptx::ld_shared_v4(slot + a0);
    w0 = v0.x; w1 = v0.y; w2 = v0.z; w3 = v0.w;
  }
  if (s2 != 0) {
    uint32_t w4 = 0, w5 = 0, w6 = 0, w7 = 0;
    if (a0 + 16 < sh + rb) {
      const uint4 v1 = ptx::ld_shared_v4(slot + a0 + 16);
      w4 = v1.x; w5 = v1.y; w6 = v1.z; w7 = v1.w;
    }
    if (s2 & 8) { w0 = w2; w1 = w3; w2 = w4; w3 = w5; w4 = w6; w5 = w7; }
    if (s2 & 4) { w0 = w1; w1 = w2; w2 = w3; w3 = w4; w4 = w5; }
    if (s2 & 2) {
      w0 = __funnelshift_r(w0, w1, 16); w1 = __funnelshift_r(w1, w2, 16);
      w2 = __funnelshift_r(w2, w3, 16); w3 = __funnelshift_r(w3, w4, 16);
    }
  }
  if (o < 0 || o + 16 > rb) {  // row edge: zero the bytes outside [0, rb)
    uint32_t w[4] = {w0, w1, w2, w3};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t m = 0;
#pragma unroll
      for (int bb = 0; bb < 4; ++bb) {
        const int oo = o + 4 * k + bb;
        if (oo >= 0 && oo < rb) m |= 0xFFu << (8 * bb);
      }
      w[k] &= m;
    }
    w0 = w[0]; w1 = w[1]; w2 = w[2]; w3 = w[3];
  }
  return make_uint4(w0, w1, w2, w3);
}

// Per-lane chunk map of the folded layout (identical for every raw row):
// chunk k of this lane = (region q', folded column w''), its byte offset in the
// raw row (src) and in the region row (dst). Computed once per warp.
struct FoldChunks {
  int n;            // chunks of this lane (<= 4; 0 = use the generic loop)
  int src[4], dst[4];
};

// Per-lane chunk map. Legacy layout: 16-byte core column q' of folded column
// w'' -> region q' (the shift region q' = Q holds core column 0 of w''+1).
// SWIZZLE_32B layout: 16-byte half h of the 32-byte K-step at in-pixel offset
// qs[qi] -> region qi, logical byte (w'' * 32 + h * 16) of the row (the
// row-dependent swizzle is applied per row in transpose_row).
__device__ __forceinline__ FoldChunks fold_chunks(const RowProd& p, const ConvArgs& a, int lane) {
  FoldChunks fc;
  const int nck = p.sw32 ? (a.nq * 2) << p.lw : p.Qr << p.lw;
  fc.n = (nck <= 128) ? (nck - lane + 31) / 32 : 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int c = lane + 32 * k;
    if (p.sw32) {
      const int w2 = c & (p.Wbox - 1);
      const int qh = c >> p.lw;  // qi * 2 + h
      const int qi = qh >> 1, h = qh & 1;
      fc.src[k] = (p.c0 + w2) * p.pix + a.qbyte[qi & 3] + h * 16;
      fc.dst[k] = qi * p.qregion_bytes + w2 * 32 + h * 16;
    } else {
      const int qq = c >> p.lw;
      const int w2 = c & (p.Wbox - 1);
      fc.src[k] = (p.c0 + w2) * p.pix + ((qq == p.Q) ? p.pix : qq * 16);
      fc.dst[k] = qq * p.lbo + w2 * 16;
    }
  }
  return fc;
}

// Transpose one staged (or zero) raw row r of the stage into the A stage at `dst`.
template <int kProd>
__device__ __forceinline__ void transpose_row(const RowProd& p, const FoldChunks& fc, const StageRows& sr, int r,
                                              bool staged, int mt, uint32_t dst, uint32_t slot, int sh, int lane) {
  const int rb = p.rb, pix = p.pix;
  const uint4 z = make_uint4(0u, 0u, 0u, 0u);
  if (kProd == 1 && fc.n > 0) {
    const uint32_t e = ptx::ld_shared_u32(p.row_tab + 4 * r);
    // legacy: region row i at i * Wbox * 16; sw32: logical row offset i * Wbox * 32, then
    // the SWIZZLE_32B XOR (16-byte half ^= address bit 7) on the 1024-aligned region
    const uint32_t rbase = dst + (e & 0xFF) * p.region_bytes + (p.sw32 ? 0u : ((e >> 8) & 0xFF) * p.Wbox * 16);
    const uint32_t rlog = p.sw32 ? ((e >> 8) & 0xFF) * p.Wbox * 32 : 0u;
    const bool fast = sh == 0 && (pix & 15) == 0 && (rb & 15) == 0;
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[k] = z;
      if (k < fc.n && staged) {
        const int o = fc.src[k];
        if (fast) {
          if (o >= 0 && o < rb) v[k] = ptx::ld_shared_v4(slot + o);
        } else {
          v[k] = raw16(slot, sh, o, rb);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k >= fc.n) continue;
      uint32_t o = fc.dst[k];
      if (p.sw32) {  // region offset + swizzled in-region address
        const uint32_t qoff = (o / p.qregion_bytes) * p.qregion_bytes;
        const uint32_t L = rlog + (o - qoff);
        o = qoff + (L ^ (((L >> 7) & 1u) << 4));
      }
      ptx::st_shared_v4(rbase + o, v[k].x, v[k].y, v[k].z, v[k].w);
    }
  } else if (kProd == 1) {
    // regions q' of residue b, region row i: chunk (q', w'') = folded pixel
    // c0 + w'' (+1 for the shift region q' = Q), core column q' % Q
    const uint32_t e = ptx::ld_shared_u32(p.row_tab + 4 * r);
    const uint32_t rbase = dst + (e & 0xFF) * p.region_bytes + ((e >> 8) & 0xFF) * p.Wbox * 16;
    const int nck = p.Qr << p.lw;
    const int wmask = p.Wbox - 1;
    // 16-byte aligned rows with 16-byte pixels: every chunk is one aligned
    // shared-memory load, wholly inside or wholly outside the row
    const bool fast = sh == 0 && (pix & 15) == 0 && (rb & 15) == 0;
#pragma unroll 4
    for (int c = lane; c < nck; c += 32) {
      const int qq = c >> p.lw;
      const int w2 = c & wmask;
      const int o = (p.c0 + w2) * pix + ((qq == p.Q) ? pix : qq * 16);
      uint4 v = z;
      if (staged) {
        if (fast) {
          if (o >= 0 && o < rb) v = ptx::ld_shared_v4(slot + o);
        } else {
          v = raw16(slot, sh, o, rb);
        }
      }
      ptx::st_shared_v4(rbase + qq * p.lbo + w2 * 16, v.x, v.y, v.z, v.w);
    }
  } else {
    // im2col: raw row (output row t of the tile, kh) feeds M rows m of that output row
    const int t = r / sr.nkh;
    const int kh = sr.kh0 + (r - t * sr.nkh);
    const long long P0 = static_cast<long long>(mt) * 128;
    const long long pr0 = (sr.g0 + t) * p.OW;  // first pixel of the output row
    const int m_lo = static_cast<int>(max(pr0, P0) - P0);
    const int m_hi = static_cast<int>(min(min(pr0 + p.OW, P0 + 128), p.total_px) - P0);
    const uint32_t kbase = dst + (kh - sr.kh0) * p.U * 4096;
    const int step = p.sw * pix;                                       // raw bytes between M rows
    const int o0 = (static_cast<int>(P0 - pr0) * p.sw - p.pw) * pix;  // raw offset of M row 0
    for (int uc = 0; uc < 2 * p.U; ++uc) {
      const uint32_t ubase = kbase + (uc >> 1) * 4096 + (uc & 1) * 2048;
#pragma unroll 4
      for (int m = m_lo + lane; m < m_hi; m += 32) {
        const uint4 v = staged ? raw16(slot, sh, o0 + m * step + uc * 16, rb) : z;
        ptx::st_shared_v4(ubase + m * 16, v.x, v.y, v.z, v.w);
      }
    }
  }
}

// ---- staged gather producer (kProd 4) ------------------------------------------
// For rows whose pitch TMA cannot address (AlexNet: 227 px x 3 ch x 2 B = 1362
// bytes, 2-byte aligned) the A stages are built from the rows themselves, with
// no workspace and no second pass over the input. The input rows of a stage
// unit are contiguous in x: warp 0 lands the whole span (its 16-byte aligned
// superset) in a raw slot with bulk copies (two slots, the next unit's copy in
// flight while this one is realigned; the L2 is prefetched a further unit
// ahead). The gather warps then realign it: each lane reads aligned 16-byte
// blocks of a row's folded window from the slot, takes its right neighbour's
// block by a warp shuffle, funnel-shifts the pair by the row's misalignment
// and stores the 16-byte core column at its place in the A layout -- the same
// shared-memory image the TMA boxes land (plan.hpp), so the MMA schedule is
// unchanged. (Reading the rows with per-lane global loads instead was bound by
// their latency: ~1.5x slower on AlexNet.) Chunk k of a row window is core
// column k % Q of folded pixel c0 + k / Q; with the shift region (Qr = Q + 1)
// core column 0 of pixel w'' + 1 is stored again as region Q of column w''.

// Input bytes [s0, s1) (relative to x, 16-byte aligned superset) holding the
// rows [oh0*s - ph, (oh0 + tps*OHt - 1)*s - ph + KH) of stage unit u, clipped
// to the image; empty when the unit lies past the batch.
__device__ __forceinline__ void unit_span(const ConvArgs& a, const RowProd& p, int u, int& n, int& oh0,
                                          long long& s0, long long& s1) {
  tile_origin<1>(a, u, 0, 0u, n, oh0);
  s0 = s1 = 0;
  if (n >= p.n_img) return;
  const int lo = max(0, oh0 * p.s - p.ph), hi = min(p.H, (oh0 + a.tps * p.OHt - 1) * p.s - p.ph + p.kh_count);
  if (hi <= lo) return;
  const long long img = static_cast<long long>(n) * p.in_img_bytes;
  s0 = (img + static_cast<long long>(lo) * p.rb) & ~15LL;
  s1 = (img + static_cast<long long>(hi) * p.rb + 15) & ~15LL;
}
struct GatherRow {
  uint4 v[4];     // this lane's aligned blocks lane + 32i of the window
  int s2;         // window misalignment in bytes (even; warp-uniform)
  uint32_t roff;  // A-stage offset of the row: residue region + region row
};

// Loads of raw row r of the stage unit at (image n, first output row oh0) from
// the raw slot holding input bytes [s0, ...). Everything but the block index
// is warp-uniform; per-block bounds are 32-bit offsets from the row start.
__device__ __forceinline__ void gather_load(const RowProd& p, int n, int oh0, int r, int lane, int nit,
                                            uint32_t slot, long long s0, GatherRow& g, bool direct) {
  const uint32_t e = ptx::ld_shared_u32(p.row_tab + 4 * r);
  const int ih = (oh0 + static_cast<int>(static_cast<int8_t>(e >> 16))) * p.s + static_cast<int>(e & 0xFF);
  g.roff = (e & 0xFF) * p.region_bytes + ((e >> 8) & 0xFF) * p.Wbox * 16;
  const bool valid = ih >= 0 && ih < p.H && n < p.n_img;
  const long long row = static_cast<long long>(n) * p.in_img_bytes + static_cast<long long>(ih) * p.rb;
  const int wrel = p.c0 * p.pix;                        // window start relative to the row (< 0: left padding)
  const int mis = static_cast<int>((row + wrel) & 15);  // (row + wrel) mod 16, wrel possibly negative
  g.s2 = mis;
  const int rel0 = wrel - mis;                          // first block, relative to the row start
  const uint32_t sb = slot + static_cast<uint32_t>(row + rel0 - s0);  // its slot address (16-byte aligned)
  const uint8_t* const gb = p.x + (row + rel0);                        // direct (a.prod 6): the block in x
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int brel = rel0 + 16 * (lane + 32 * i);
    // only blocks holding row bytes are read (an aligned block never crosses a page)
    const bool ok = valid && i < nit && brel > -16 && brel < p.rb;
    if (direct)
      g.v[i] = ok ? ptx::ld_global_nc_v4(gb + 16 * (lane + 32 * i)) : make_uint4(0u, 0u, 0u, 0u);
    else
      g.v[i] = ok ? ptx::ld_shared_v4(sb + 16 * (lane + 32 * i)) : make_uint4(0u, 0u, 0u, 0u);
  }
}

// Bytes [s2, s2 + 16) of the 32-byte pair (a, b), s2 = 4*Q4 + (0 | 2).
template <int Q4>
__device__ __forceinline__ uint4 realign(const uint4& a, const uint4& b, uint32_t sh) {
  const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  return make_uint4(__funnelshift_r(w[Q4], w[Q4 + 1], sh), __funnelshift_r(w[Q4 + 1], w[Q4 + 2], sh),
                    __funnelshift_r(w[Q4 + 2], w[Q4 + 3], sh), __funnelshift_r(w[Q4 + 3], w[Q4 + 4], sh));
}

// Zero the chunk bytes outside the row: keep [lo, hi) of the 16.
__device__ __forceinline__ uint4 edge_mask(uint4 c, int lo, int hi) {
  uint32_t w[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int a = min(max(lo - 4 * k, 0), 4), b = min(max(hi - 4 * k, 0), 4);
    const uint32_t keep_hi = (b >= 4) ? 0xFFFFFFFFu : ((1u << (8 * b)) - 1u);
    const uint32_t drop_lo = (a >= 4) ? 0xFFFFFFFFu : ((1u << (8 * a)) - 1u);
    w[k] &= keep_hi & ~drop_lo;
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

template <int Q4, bool kShift>
__device__ __forceinline__ void gather_store_q(const GatherRow& g, const uint4 (&t)[4], uint32_t rbase, int lane,
                                               const int (&d1)[4], const int (&d2)[4], unsigned edge, int o0, int rb) {
  const uint32_t sh = static_cast<uint32_t>(g.s2 & 3) * 8;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (d1[i] < 0 && (!kShift || d2[i] < 0)) continue;
    // right neighbour block: lane + 1's block i, or (lane 31) lane 0's block i + 1
    const uint4 nx = (lane == 31) ? (i < 3 ? t[i + 1] : make_uint4(0u, 0u, 0u, 0u)) : t[i];
    uint4 c = realign<Q4>(g.v[i], nx, sh);
    if ((edge >> i) & 1u) {  // chunk at a row edge (per lane, row independent)
      const int o = o0 + 512 * i;
      c = edge_mask(c, -o, rb - o);
    }
    if (d1[i] >= 0) ptx::st_shared_v4(rbase + d1[i], c.x, c.y, c.z, c.w);
    if (kShift && d2[i] >= 0) ptx::st_shared_v4(rbase + d2[i], c.x, c.y, c.z, c.w);
  }
}

__device__ __forceinline__ uint32_t shfl_next(uint32_t v, int lane) {
  return __shfl_sync(0xffffffffu, v, (lane + 1) & 31);
}

// Realign the row's blocks into 16-byte chunks and store them into the A stage.
template <bool kShift>
__device__ __forceinline__ void gather_store(const GatherRow& g, uint32_t stage, int lane, const int (&d1)[4],
                                             const int (&d2)[4], unsigned edge, int o0, int rb) {
  uint4 t[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    t[i] = make_uint4(shfl_next(g.v[i].x, lane), shfl_next(g.v[i].y, lane), shfl_next(g.v[i].z, lane),
                      shfl_next(g.v[i].w, lane));
  const uint32_t rbase = stage + g.roff;
  switch (g.s2 >> 2) {  // warp-uniform
    case 0: gather_store_q<0, kShift>(g, t, rbase, lane, d1, d2, edge, o0, rb); break;
    case 1: gather_store_q<1, kShift>(g, t, rbase, lane, d1, d2, edge, o0, rb); break;
    case 2: gather_store_q<2, kShift>(g, t, rbase, lane, d1, d2, edge, o0, rb); break;
    default: gather_store_q<3, kShift>(g, t, rbase, lane, d1, d2, edge, o0, rb); break;
  }
}

template <int kKind, int kPair>
__device__ __forceinline__ void issue_mma(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  if constexpr (kPair == 2) {
    static_assert(kKind == 0, "pair mode runs kind::f16");
    ptx::mma_pair(d, adesc, bdesc, idesc, acc);
  } else {
    ptx::mma<kKind>(d, adesc, bdesc, idesc, acc);
  }
}
template <int kPair>
__device__ __forceinline__ void commit_to(uint32_t bar) {
  if constexpr (kPair == 2) ptx::mma_commit_pair(bar, 0x3);  // both CTAs of the pair
  else ptx::mma_commit(bar);
}
// Accumulator-drained signal. Single CTA: every thread arrives on its own
// CTA's barrier. Pair: one remote arrive per warp (after every lane's
// tcgen05.wait::ld) on the leader's barrier.
template <int kPair>
__device__ __forceinline__ void arrive_at(uint32_t bar) {
  if constexpr (kPair == 2) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) ptx::mbar_arrive_cluster(bar);
  } else {
    ptx::mbar_arrive(bar);
  }
}

// kPair = 2: a cluster of two CTAs (one per SM of a TPC) runs cta_group::2
// MMAs -- M = 256 (each CTA's 128-row tile), each CTA holding half of every B
// block, so the per-SM shared-memory operand traffic drops by the B half.
// kMc = 1: the two N-tiles of a plan run as a 2-CTA cluster walking the same
// M tiles; each CTA issues the TMA boxes of every other residue with
// .multicast::cluster so both receive the whole A stage and each SM's TMA
// unit issues half of the pieces; a stage is refilled only after both CTAs'
// MMAs released it (multicast commits, empty barriers of count 2).
template <int kKind, typename OutT, int CH, int kProd, int kPair = 1, int kMc = 0>
__global__ void __launch_bounds__(kProd == 0 ? 320 : 320 + 32 * (kProd == 4 ? kGatherWarps4 : (kProd == 5 ? kGatherWarps5 : kGatherWarps)), 1)
    conv_fold_kernel(const __grid_constant__ ConvArgs a, const __grid_constant__ TmaMaps maps) {
  using namespace ptx;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t bar_full = base;          // [stages] x 8 B
  const uint32_t bar_empty = base + 64;    // [stages] x 8 B
  const uint32_t bar_tfull = base + 384;      // [n_acc <= 4] x 8 B: accumulator written
  const uint32_t bar_tempty = base + 416;     // [n_acc] x 8 B: lower half of the accumulator drained
  const uint32_t bar_tempty_hi = base + 448;  // [n_acc] x 8 B: upper half drained
  const uint32_t bar_bpeer = base + 184;      // pair: the peer's B half landed (leader's barrier)
  const uint32_t bar_b = base + 160;
  const uint32_t bar_raw_full = base + 1024;   // [raw_slots <= 32] x 8 B
  const uint32_t bar_raw_empty = base + 1280;  // [raw_slots <= 32] x 8 B (control area: kCtrlBytes)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + 192);

  // warp index via shuffle so the compiler knows it is warp-uniform (keeps the
  // MMA issuer's operands in uniform registers)
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const uint32_t rank = (kPair == 2) ? cluster_ctarank() : 0u;  // 0: pair leader (issues the MMAs)
  const uint32_t mrank = kMc ? cluster_ctarank() : 0u;           // multicast cluster: this CTA's residue half
  const int cl = static_cast<int>(blockIdx.x) / kPair;           // cluster (or CTA) index
  const int ntile = cl % a.n_tiles;
  const int local = cl / a.n_tiles;                               // first M-tile unit of this CTA
  const int ncols = a.nt_cols[ntile];
  const int col0 = a.nt_col0[ntile];
  if (threadIdx.x == 0) tl_mark(a, gbase, 0);  // entry

  if (kProd == 1 || kProd == 4)  // folded stage-row table of the row producers (b | i << 8 | a << 16)
    for (int r = threadIdx.x; r < a.rows_per_stage; r += blockDim.x)
      reinterpret_cast<uint32_t*>(gbase + 768)[r] = static_cast<uint32_t>(static_cast<uint8_t>(a.row_b[r])) |
                                                    (static_cast<uint32_t>(static_cast<uint8_t>(a.row_i[r])) << 8) |
                                                    (static_cast<uint32_t>(static_cast<uint8_t>(a.row_a[r])) << 16);
  if (threadIdx.x == 0) {
    for (int i = 0; i < a.stages; ++i) {
      // TMA: one expect_tx; rows: one arrive per transposer / gather warp
      mbar_init(bar_full + 8 * i, (kProd == 0 || kProd == 5) ? 1 : (kProd == 4 ? kGatherWarps4 : kGatherWarps));
      mbar_init(bar_empty + 8 * i, (kMc && !prof(a, 0x2000)) ? 2 : 1);  // multicast: both CTAs' MMAs release the stage
    }
    for (int i = 0; i < a.n_acc; ++i) {
      mbar_init(bar_tfull + 8 * i, 1);
      // every epilogue thread arrives (pair: one arrive per warp of both CTAs, on the leader's)
      mbar_init(bar_tempty + 8 * i, kPair == 2 ? 16 : (a.epi_pp ? 128 : 256));  // ping-pong: one warp group per tile
      mbar_init(bar_tempty_hi + 8 * i, kPair == 2 ? 16 : (a.epi_pp ? 128 : 256));
    }
    mbar_init(bar_b, 1);
    mbar_init(bar_bpeer, 1);
    for (int i = 0; i < a.raw_slots; ++i) {
      // ring (kProd 5): every gather warp fills the slot, the MMA issuer frees it
      // (multicast cluster: both CTAs' gather warps fill the shared slot, both MMA issuers free it)
      mbar_init(bar_raw_full + 8 * i, (kProd == 5 && kMc) ? 2 : 1);
      mbar_init(bar_raw_empty + 8 * i, kProd == 4 ? kGatherWarps4 : ((kProd == 5 && kMc) ? 2 : 1));
    }
    fence_barrier_init();
  }
  if ((kProd == 0 || kProd == 5) && warp == 0 && lane == 0) {
    for (int b = 0; b < a.s; ++b)
      if ((a.res_mask >> b) & 1u) {
        prefetch_tmap(&maps.in[b]);
        if (a.shift_box_bytes) prefetch_tmap(&maps.in_shift[b]);
      }
  }
  if (warp == 1) {
    if constexpr (kPair == 2) tmem_alloc_pair(smem_u32(tmem_slot), a.tmem_cols);
    else tmem_alloc(smem_u32(tmem_slot), a.tmem_cols);
  }
  tc_fence_before();
  if constexpr (kPair == 2 || kMc) cluster_sync();  // the peer's barriers are initialised before remote use
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Programmatic dependent launch: everything above (launch, barrier init, TMEM
  // allocation, tensor-map prefetch) overlaps the previous grid's tail, and so
  // does the producer's bulk copy of the packed filter (B): every other global
  // access -- x, the workspace, the bias, every store of y -- comes after
  // griddepcontrol.wait in the thread that makes it. B is written only by the
  // pack kernel; the first launch after any pack runs without the PDL
  // attribute (host side, conv_fold.cu), so that B is complete when read.
  // The next grid may start its own prologue from here on.
  if (threadIdx.x == 0) tl_mark(a, gbase, 1);  // prologue done
  griddep_launch_dependents();
  if (warp >= 2) griddep_wait();  // epilogue and gather warps (warp 0: after B; warp 1 touches no global memory)

  if (kProd == 5 && warp >= 10) {
    // ===================== L2-ring gather warps (warps 10..17) =====================
    // Stage unit it of this CTA: the ring_rows input rows from (oh0 + amin_min)*s
    // are read with coalesced 16-byte loads of their aligned blocks, realigned
    // (neighbour block by shuffle, funnel shift by the row's misalignment) and
    // stored as re-pitched rows (16-byte pitch, zero tail) into ring slot it % R
    // of this CTA. The slot is handed to the TMA producer through an mbarrier
    // after a generic -> async proxy fence; the MMA issuer frees it once the
    // stage built from it has landed. Slots are rewritten every R units, so
    // the ring stays in L2: x is read from HBM once, nothing extra is written.
    // In the multicast N-tile cluster the two CTAs share one ring (per
    // cluster): each re-pitches every other row of the slot and signals both.
    const int gw = warp - 10;
    constexpr int kStep = kMc ? 2 : 1;  // CTAs sharing the slot
    constexpr int P = kGatherWarps5;
    const uint8_t* const x = reinterpret_cast<const uint8_t*>(opq64(reinterpret_cast<long long>(a.x)));
    const long long img_b = opq64(a.in_img_bytes);
    const int rb = opq(static_cast<int>(a.in_row_bytes)), rp = opq(a.ring_rowpitch);
    const int nblk = rp >> 4;  // 16-byte blocks of a re-pitched row
    const int SR = opq(a.ring_rows), R = opq(a.raw_slots), H = opq(a.H), nimg = opq(a.n_img), s = opq(a.s);
    const int amin0 = opq(a.amin_min);
    const long long slot_b = opq64(a.ring_slot_bytes);
    uint8_t* const ring = a.ring + static_cast<long long>(blockIdx.x / kStep) * R * slot_b;
    // L2 prefetch of the input span of the unit two ahead (one bulk prefetch:
    // a unit's rows are contiguous in x), so the row loads hit L2
    const RowProd rpf = row_prod(a, 0u);
    auto prefetch_unit = [&](int u) {
      int n, oh0;
      long long s0, s1;
      unit_span(a, rpf, u, n, oh0, s0, s1);
      if (s1 > s0) prefetch_l2_bulk(x + s0, static_cast<uint32_t>(s1 - s0));
    };
    const bool pf = gw == 0 && lane == 0;
    // profiling (PROFILE builds): 0x8000 the gather warps skip their row loads (zeros), 0x10000 the proxy fence
    const bool no_ld = prof(a, 0x8000), no_fence = prof(a, 0x10000);
    if (pf)
      for (int u = local; u < a.num_units && u < local + 2 * a.unit_stride; u += a.unit_stride) prefetch_unit(u);
    int slot = 0;
    uint32_t round = 0;
    // profiling (0x80000, CTA 0, gather warp 0): cycles waiting for a free slot, loading + storing, fencing
    const bool dbg = prof(a, 0x80000) && blockIdx.x == 0 && gw == 0 && lane == 0;
    long long t_empty = 0, t_rows = 0, t_fence = 0, t_arrive = 0, t_ld = 0, t0 = 0, t_all = dbg ? clock64() : 0;
    for (int u = local; u < a.num_units; u += a.unit_stride) {
      if (pf && u + 2 * a.unit_stride < a.num_units) prefetch_unit(u + 2 * a.unit_stride);
      if (dbg) t0 = clock64();
      if constexpr (kMc) mbar_wait_cluster(bar_raw_empty + 8 * slot, (round & 1u) ^ 1u);
      else mbar_wait(bar_raw_empty + 8 * slot, (round & 1u) ^ 1u);
      if (dbg) { const long long t1 = clock64(); t_empty += t1 - t0; t0 = t1; }
      int n, oh0;
      tile_origin<1>(a, u, 0, 0u, n, oh0);
      const int row0 = (oh0 + amin0) * s;
      uint8_t* const dslot = ring + slot * slot_b;
      for (int j0 = static_cast<int>(mrank) + kStep * gw; j0 < SR; j0 += 3 * kStep * P) {  // three rows in flight per warp
        uint4 v[3][4];
        int mis[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const int j = j0 + q * kStep * P, ih = row0 + j;
          const bool ok = j < SR && ih >= 0 && ih < H && n < nimg && !no_ld;
          const long long rs = static_cast<long long>(n) * img_b + static_cast<long long>(ih) * rb;
          mis[q] = ok ? static_cast<int>(rs & 15) : 0;
          const uint8_t* blk = x + (rs - mis[q]);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int kb = lane + 32 * i;  // aligned block kb of the row (blocks holding row bytes only)
            v[q][i] = (ok && kb <= nblk && 16 * kb - mis[q] < rb) ? ld_global_nc_v4(blk + 16 * kb)
                                                                  : make_uint4(0u, 0u, 0u, 0u);
          }
        }
#if WFB_PROFILE
        if (dbg) {  // wait for this batch's loads (a volatile move of the last block), then read the clock
          const long long tl0 = clock64();
          uint32_t dep;
          asm volatile("mov.b32 %0, %1;" : "=r"(dep) : "r"(v[2][2].x ^ v[0][0].y));
          t_ld += clock64() - tl0 + (dep & 0);
        }
#endif
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const int j = j0 + q * kStep * P;
          if (j >= SR) break;
          uint4 t[4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            t[i] = make_uint4(shfl_next(v[q][i].x, lane), shfl_next(v[q][i].y, lane), shfl_next(v[q][i].z, lane),
                              shfl_next(v[q][i].w, lane));
          const uint32_t sh = static_cast<uint32_t>(mis[q] & 3) * 8;
          uint8_t* const drow = dslot + static_cast<long long>(j) * rp;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int ob = lane + 32 * i;  // output block: bytes [16 ob, 16 ob + 16) of the re-pitched row
            if (ob >= nblk) continue;
            const uint4 nx = (lane == 31) ? (i < 3 ? t[i + 1] : make_uint4(0u, 0u, 0u, 0u)) : t[i];
            uint4 c;
            switch (mis[q] >> 2) {  // warp-uniform
              case 0: c = realign<0>(v[q][i], nx, sh); break;
              case 1: c = realign<1>(v[q][i], nx, sh); break;
              case 2: c = realign<2>(v[q][i], nx, sh); break;
              default: c = realign<3>(v[q][i], nx, sh); break;
            }
            if (16 * ob + 16 > rb) c = edge_mask(c, 0, rb - 16 * ob);  // zero tail past W*C
            st_global_v4(drow + 16 * ob, c);
          }
        }
      }
      if (dbg) { const long long t1 = clock64(); t_rows += t1 - t0; t0 = t1; }
      if (!no_fence) fence_proxy_async_global();  // generic-proxy stores -> visible to the TMA reads of the slot
      named_bar_sync(2, 32 * P);  // every gather warp's rows of the slot are written and fenced
      if (dbg) t_fence += clock64() - t0;
      if (gw == 0 && lane == 0) {  // one arrival per CTA (one release instead of one per warp)
        if constexpr (kMc) {  // both CTAs' producers load from the slot (release at cluster scope)
          mbar_arrive_cluster(mapa(bar_raw_full + 8 * slot, 0));
          mbar_arrive_cluster(mapa(bar_raw_full + 8 * slot, 1));
        } else {
          mbar_arrive(bar_raw_full + 8 * slot);
        }
      }
      if (dbg) { const long long t1 = clock64(); t_arrive += t1 - t0; }
      if (++slot == R) { slot = 0; ++round; }
    }
#if WFB_PROFILE
    if (dbg)
      printf("ring gather warp0 cta0: %lld cycles: wait free slot %lld, rows (load+realign+store) %lld (of which load "
             "latency %lld), fence+bar %lld, arrive %lld\n",
             clock64() - t_all, t_empty, t_rows, t_ld, t_fence, t_arrive);
#endif
  } else if (kProd == 4 && warp >= 10) {
    // ===================== direct gather producer (warps 10..17) =====================
    const RowProd rp = row_prod(a, base + 768);
    const int gw = warp - 10;
    // this lane's chunks (row independent): region offsets of core column k % Q of
    // folded column k / Q, and of its shift-region copy (-1: not stored)
    int d1[4], d2[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = lane + 32 * i;
      const int q = k % rp.Q, w2 = k / rp.Q;
      d1[i] = (w2 < rp.Wbox) ? q * rp.lbo + w2 * 16 : -1;
      d2[i] = (rp.Qr > rp.Q && q == 0 && w2 >= 1 && w2 <= rp.Wbox) ? rp.Q * rp.lbo + (w2 - 1) * 16 : -1;
    }
    const int nit = (rp.Q * rp.Wbox + 2 + 31) / 32;  // block iterations per row (<= 4, planner-checked)
    const bool has_shift = rp.Qr > rp.Q;              // shift region (uniform)
    // chunks at a row edge (row-relative offset o outside [0, rb - 16]): byte-masked
    const int o0 = rp.c0 * rp.pix + 16 * lane;
    unsigned edge = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int o = o0 + 512 * i;
      if (o < 0 || o + 16 > rp.rb) edge |= 1u << i;
    }
    const int rps = rp.rows_per_stage;
    const int nstages = a.stages, stage_bytes = a.stage_bytes, stride = a.unit_stride, units = a.num_units;
    const uint32_t a_base = base + a.off_a, raw_base = base + a.off_raw;
    GatherRow g0, g1;
    constexpr int P = kGatherWarps4;
    // a.prod 6 (direct): no raw slots -- rows are read straight from x, whose
    // unit spans gather warp 0 prefetches into L2 two units ahead
    const bool direct = a.prod == 6;
    const bool pf = direct && gw == 0 && lane == 0;
    auto prefetch_unit = [&](int u) {
      int n, oh0;
      long long s0, s1;
      unit_span(a, rp, u, n, oh0, s0, s1);
      if (s1 > s0) prefetch_l2_bulk(rp.x + s0, static_cast<uint32_t>(s1 - s0));
    };
    if (pf)
      for (int u = local; u < units && u < local + 2 * stride; u += stride) prefetch_unit(u);
    int it = 0;
    for (int u = local; u < units; u += stride, ++it) {
      const int stage = it % nstages;
      const uint32_t round = static_cast<uint32_t>(it / nstages);
      const int rs = it & 1;  // raw slot of this unit
      int n, oh0;
      long long s0, s1;
      unit_span(a, rp, u, n, oh0, s0, s1);
      const uint32_t slot = raw_base + rs * rp.raw_slot_bytes;
      if (direct) {
        if (pf && u + 2 * stride < units) prefetch_unit(u + 2 * stride);
      } else {
        mbar_wait(bar_raw_full + 8 * rs, static_cast<uint32_t>(it >> 1) & 1u);
      }
      // two rows in flight: load one while the other is realigned and stored
      int r = gw;
      if (r < rps) gather_load(rp, n, oh0, r, lane, nit, slot, s0, g0, direct);
      if (r + P < rps) gather_load(rp, n, oh0, r + P, lane, nit, slot, s0, g1, direct);
      mbar_wait(bar_empty + 8 * stage, (round & 1u) ^ 1u);
      const uint32_t dst = a_base + stage * stage_bytes;
      auto store = [&](const GatherRow& g) {
        if (has_shift) gather_store<true>(g, dst, lane, d1, d2, edge, o0, rp.rb);
        else gather_store<false>(g, dst, lane, d1, d2, edge, o0, rp.rb);
      };
      for (; r < rps; r += 2 * P) {
        store(g0);
        if (r + 2 * P < rps) gather_load(rp, n, oh0, r + 2 * P, lane, nit, slot, s0, g0, direct);
        if (r + P < rps) {
          store(g1);
          if (r + 3 * P < rps) gather_load(rp, n, oh0, r + 3 * P, lane, nit, slot, s0, g1, direct);
        }
      }
      __syncwarp();
      if (lane == 0 && !direct) mbar_arrive(bar_raw_empty + 8 * rs);  // the slot's rows are consumed
      fence_proxy_async_smem();  // generic-proxy stores -> visible to tcgen05
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_full + 8 * stage);
    }
  } else if (kProd == 4 && warp == 0) {
    // B operand, then each stage unit's raw input span into the two raw slots
    if (elect_one()) {
      const uint8_t* gb = reinterpret_cast<const uint8_t*>(a.nt_bsrc[ntile]);
      const int bb = a.nt_bbytes[ntile];
      mbar_arrive_expect_tx(bar_b, static_cast<uint32_t>(bb));
      for (int off = 0; off < bb; off += 32768)
        bulk_g2s(base + a.off_b + off, gb + off, static_cast<uint32_t>(min(32768, bb - off)), bar_b);
      griddep_wait();  // B overlaps the previous grid; x / workspace come after the wait
      const RowProd rp = row_prod(a, base + 768);
      const int stride = a.unit_stride, units = a.num_units;
      auto prefetch_unit = [&](int u) {  // L2 prefetch of a later unit's span
        int n, oh0;
        long long s0, s1;
        unit_span(a, rp, u, n, oh0, s0, s1);
        if (s1 > s0) prefetch_l2_bulk(rp.x + s0, static_cast<uint32_t>(s1 - s0));
      };
      for (int u = local; u < units && u < local + 2 * stride && a.prod != 6; u += stride) prefetch_unit(u);
      int it = 0;
      for (int u = local; u < units && a.prod != 6; u += stride, ++it) {  // (6: the gather warps read x)
        const int rs = it & 1;
        mbar_wait(bar_raw_empty + 8 * rs, (static_cast<uint32_t>(it >> 1) & 1u) ^ 1u);
        if (u + 2 * stride < units) prefetch_unit(u + 2 * stride);
        int n, oh0;
        long long s0, s1;
        unit_span(a, rp, u, n, oh0, s0, s1);
        const uint32_t bytes = static_cast<uint32_t>(s1 - s0);
        const uint32_t slot = base + a.off_raw + rs * rp.raw_slot_bytes;
        mbar_arrive_expect_tx(bar_raw_full + 8 * rs, bytes);
        for (uint32_t off = 0; off < bytes; off += 32768)
          bulk_g2s(slot + off, rp.x + s0 + off, min(32768u, bytes - off), bar_raw_full + 8 * rs);
      }
    }
    __syncwarp();
  } else if ((kProd == 1 || kProd == 2) && (warp == 0 || warp >= 10)) {
    // ===================== row-staged producer =====================
    // warp 0 (one lane): B operand, then one bulk copy per raw input row into
    // the slot ring; warps 10..12: transpose staged rows into the A stages.
    const uint32_t ring = base + a.off_raw;
    const RowProd rp = row_prod(a, base + 768);
    const FoldChunks fc = fold_chunks(rp, a, lane);
    if (warp == 0) {
      if (elect_one()) {
        const uint8_t* gb = reinterpret_cast<const uint8_t*>(a.nt_bsrc[ntile]);
        const int bb = a.nt_bbytes[ntile];
        mbar_arrive_expect_tx(bar_b, static_cast<uint32_t>(bb));
        for (int off = 0; off < bb; off += 32768)
          bulk_g2s(base + a.off_b + off, gb + off, static_cast<uint32_t>(min(32768, bb - off)), bar_b);
      griddep_wait();  // B overlaps the previous grid; x / workspace come after the wait
        int slot_it = 0;
        const bool no_loads = prof(a, 0x1000);
        for (int mt = local; mt < a.num_units; mt += a.unit_stride)  // stage units (= M tiles unless tps 2)
          for (int ks = 0; ks < rp.ksplit; ++ks) {
            const StageRows sr = stage_rows<kProd>(a, rp, mt, ks);
            for (int r = 0; r < sr.count; ++r) {  // every row takes a slot; padding rows carry no bytes
              int n, ih;
              const bool staged = stage_row<kProd>(rp, sr, r, n, ih) && !no_loads;
              const int slot = slot_it & (kRawSlots - 1);
              const uint32_t round = static_cast<uint32_t>(slot_it) / kRawSlots;
              ++slot_it;
              mbar_wait(bar_raw_empty + 8 * slot, (round & 1u) ^ 1u);
              if (!staged) {
                mbar_arrive(bar_raw_full + 8 * slot);
                continue;
              }
              const uintptr_t src = reinterpret_cast<uintptr_t>(rp.x + n * rp.in_img_bytes + static_cast<long long>(ih) * rp.rb);
              const uintptr_t s0 = src & ~static_cast<uintptr_t>(15);
              const uintptr_t s1 = (src + rp.rb + 15) & ~static_cast<uintptr_t>(15);
              const uint32_t bytes = static_cast<uint32_t>(s1 - s0);
              mbar_arrive_expect_tx(bar_raw_full + 8 * slot, bytes);
              bulk_g2s(ring + slot * rp.raw_slot_bytes, reinterpret_cast<const void*>(s0), bytes, bar_raw_full + 8 * slot);
            }
          }
      }
      __syncwarp();
    } else {
      const int tw = warp - 10;  // transposer 0..kGatherWarps-1
      const bool dbg = prof(a, 0x8000) && blockIdx.x == 0 && tw == 0 && lane == 0;
      long long t_empty = 0, t_full = 0, t_work = 0, t_fence = 0, t0 = 0;
      int it = 0, slot_it = 0;
      const bool no_loads = prof(a, 0x1000);
      const int nstages = a.stages, stage_bytes = a.stage_bytes;
      const uint32_t a_base = base + a.off_a;
      for (int mt = local; mt < a.num_units; mt += a.unit_stride) {  // stage units
        for (int ks = 0; ks < rp.ksplit; ++ks, ++it) {
          const int stage = it % nstages;
          const uint32_t round = static_cast<uint32_t>(it / nstages);
          const StageRows sr = stage_rows<kProd>(a, rp, mt, ks);
          if (dbg) t0 = clock64();
          mbar_wait(bar_empty + 8 * stage, (round & 1u) ^ 1u);
          if (dbg) t_empty += clock64() - t0;
          const uint32_t dst = a_base + stage * stage_bytes;
          for (int r = tw; r < sr.count; r += kGatherWarps) {  // rows dealt round-robin to the transposers
            int n, ih;
            const bool staged = stage_row<kProd>(rp, sr, r, n, ih) && !no_loads;
            const int slot = (slot_it + r) & (kRawSlots - 1);
            if (dbg) t0 = clock64();
            mbar_wait(bar_raw_full + 8 * slot, (static_cast<uint32_t>(slot_it + r) / kRawSlots) & 1u);
            if (dbg) { const long long t1 = clock64(); t_full += t1 - t0; t0 = t1; }
            const uintptr_t src = reinterpret_cast<uintptr_t>(rp.x + n * rp.in_img_bytes + static_cast<long long>(ih) * rp.rb);
            transpose_row<kProd>(rp, fc, sr, r, staged, mt, dst, ring + slot * rp.raw_slot_bytes,
                          static_cast<int>(src & 15u), lane);
            __syncwarp();
            if (dbg) t_work += clock64() - t0;
            if (lane == 0) mbar_arrive(bar_raw_empty + 8 * slot);
          }
          slot_it += sr.count;
          if (dbg) t0 = clock64();
          if (!prof(a, 0x10000)) fence_proxy_async_smem();  // generic-proxy stores -> visible to tcgen05
          __syncwarp();
          if (dbg) t_fence += clock64() - t0;
          if (lane == 0) mbar_arrive(bar_full + 8 * stage);
        }
      }
#if WFB_PROFILE
      if (dbg) printf("transposer0 cta0: fence %lld cycles\n", t_fence);
      if (dbg) printf("transposer0 cta0: stages %d  wait-empty %lld  wait-row %lld  transpose %lld cycles\n", it,
                      t_empty, t_full, t_work);
#endif
    }
  } else if (warp == 0) {
    // ===================== TMA producer (one elected lane) =====================
    if (elect_one()) {
      const int bb = a.nt_bbytes[ntile];  // this CTA's B bytes (a half per CTA in pair mode)
      const uint8_t* gb = reinterpret_cast<const uint8_t*>(a.nt_bsrc[ntile]) + rank * bb;
      mbar_arrive_expect_tx(bar_b, static_cast<uint32_t>(bb));
      for (int off = 0; off < bb; off += 32768)
        bulk_g2s(base + a.off_b + off, gb + off, static_cast<uint32_t>(min(32768, bb - off)), bar_b);
      tl_mark(a, gbase, 2);  // B issued
      griddep_wait();  // B overlaps the previous grid; x / workspace come after the wait
      tl_mark(a, gbase, 3);  // previous grid done
      if (kPair == 2 && rank != 0) {  // tell the leader's MMA issuer that our B half landed
        mbar_wait(bar_b, 0);
        mbar_arrive_cluster(mapa(bar_bpeer, 0));
      }
      const uint32_t tx = static_cast<uint32_t>((a.box_bytes + a.shift_box_bytes) * __popc(a.res_mask));
      int it = 0;
      int rslot = 0;  // kProd 5: ring slot of this unit
      uint32_t rround = 0;
      const bool pdbg = prof(a, 0x80000) && blockIdx.x == 0;
      long long p_ring = 0, p_stage = 0, p0 = 0, p_all = pdbg ? clock64() : 0;
      // profiling (0x800000, with 0x600000): the producer sits the launch out too
      for (int u = prof(a, 0x800000) ? a.num_units : local; u < a.num_units; u += a.unit_stride, ++it) {
        const int stage = it % a.stages;
        const uint32_t round = static_cast<uint32_t>(it / a.stages);
        int slot_idx = 0;  // kProd 5: the slot's index in the ring tensor maps
        if constexpr (kProd == 5) {
          // the gather warps (of both CTAs in the multicast cluster) re-pitched the unit's rows
          if (pdbg) p0 = clock64();
          if constexpr (kMc) mbar_wait_cluster(bar_raw_full + 8 * rslot, rround & 1u);
          else mbar_wait(bar_raw_full + 8 * rslot, rround & 1u);
          if (pdbg) p_ring += clock64() - p0;
          slot_idx = static_cast<int>(blockIdx.x) / (kMc ? 2 : 1) * a.raw_slots + rslot;
          if (++rslot == a.raw_slots) { rslot = 0; ++rround; }
        }
        if (pdbg) p0 = clock64();
        mbar_wait(bar_empty + 8 * stage, (round & 1u) ^ 1u);
        if (pdbg) p_stage += clock64() - p0;
        // pair: both CTAs' boxes complete on the leader's full barrier
        const uint32_t fbar = (kPair == 2) ? mapa(bar_full + 8 * stage, 0) : bar_full + 8 * stage;
        int n, oh0;
        tile_origin<kPair>(a, u, 0, rank, n, oh0);  // the stage covers tiles 0..tps-1 from here
        const uint32_t dst = base + a.off_a + stage * a.stage_bytes;
        if (prof(a, 0x1000)) {  // profiling: no A loads (stage contents stale)
          if (rank == 0) mbar_arrive(bar_full + 8 * stage);
          continue;
        }
        // profiling only: 0x20000 drops the shift boxes, 0x40000 loads residue 0 only
        const bool dbg_noshift = prof(a, 0x20000), dbg_oneres = prof(a, 0x40000);
        uint32_t txs = tx;
        if (dbg_noshift || dbg_oneres) {
          txs = 0;
          for (int b = 0; b < a.s; ++b)
            if (((a.res_mask >> b) & 1u) && !(dbg_oneres && b != __ffs(a.res_mask) - 1))
              txs += a.box_bytes + (dbg_noshift ? 0 : a.shift_box_bytes);
        }
        if (rank == 0) mbar_arrive_expect_tx(bar_full + 8 * stage, txs * kPair);
        const bool mc_self = prof(a, 0x2000);  // profiling: every CTA loads every residue into itself only
        if (a.sw32) {  // one SWIZZLE_32B box of 32-byte K-step pieces per (residue, in-pixel offset)
          for (int b = 0, j = 0; b < a.s; ++b) {
            if (!((a.res_mask >> b) & 1u)) continue;
            if (kMc && !mc_self && ((j++ & 1) != static_cast<int>(mrank))) continue;  // the peer multicasts it
            for (int qi = 0; qi < a.nq; ++qi) {
              const uint32_t dq = dst + b * a.region_bytes + qi * a.qregion_bytes;
              if constexpr (kMc)
                tma_load_4d_mc(dq, &maps.in[b], a.qcoord[qi], a.c0, oh0 + a.amin[b], n, fbar,
                               mc_self ? static_cast<uint16_t>(1u << mrank) : static_cast<uint16_t>(0x3));
              else if constexpr (kPair == 2)
                tma_load_4d_pair(dq, &maps.in[b], a.qcoord[qi], a.c0, oh0 + a.amin[b], n, fbar);
              else
                tma_load_4d(dq, &maps.in[b], a.qcoord[qi], a.c0, oh0 + a.amin[b], n, fbar);
            }
          }
          continue;
        }
        for (int b = 0, j = 0; b < a.s; ++b) {
          if (!((a.res_mask >> b) & 1u)) continue;
          if (dbg_oneres && b != __ffs(a.res_mask) - 1) continue;
          if (kMc && !mc_self && ((j++ & 1) != static_cast<int>(mrank))) continue;  // the peer multicasts this residue
          if constexpr (kMc) {
            const uint16_t mask = mc_self ? static_cast<uint16_t>(1u << mrank) : static_cast<uint16_t>(0x3);
            // kProd 5: the cluster's ring slot (rows from slot row (amin[b] - amin_min)*s + b)
            const int rrow = (kProd == 5) ? a.amin[b] - a.amin_min : oh0 + a.amin[b];
            const int img = (kProd == 5) ? slot_idx : n;
            if (kProd != 5 && a.planes_e2) {  // core-column planes: {folded-col run, row, plane, image}
              tma_load_4d_mc(dst + b * a.region_bytes, &maps.in[b], a.c0 * a.planes_e2, rrow, 0, img, fbar, mask);
              if (a.shift_box_bytes && !dbg_noshift)
                tma_load_4d_mc(dst + b * a.region_bytes + a.shift_off, &maps.in_shift[b], (a.c0 + 1) * a.planes_e2,
                               rrow, 0, img, fbar, mask);
              continue;
            }
            tma_load_5d_mc(dst + b * a.region_bytes, &maps.in[b], 0, a.c0, rrow, 0, img, fbar, mask);
            if (a.shift_box_bytes && !dbg_noshift)
              tma_load_5d_mc(dst + b * a.region_bytes + a.shift_off, &maps.in_shift[b], 0, a.c0 + 1, rrow, 0, img,
                             fbar, mask);
          } else if constexpr (kPair == 2) {
            tma_load_5d_pair(dst + b * a.region_bytes, &maps.in[b], 0, a.c0, oh0 + a.amin[b], 0, n, fbar);
            if (a.shift_box_bytes && !dbg_noshift)
              tma_load_5d_pair(dst + b * a.region_bytes + a.shift_off, &maps.in_shift[b], 0, a.c0 + 1,
                               oh0 + a.amin[b], 0, n, fbar);
          } else if constexpr (kProd == 5) {  // ring slot: residue-b rows from slot row (amin[b] - amin_min)*s + b
            tma_load_5d(dst + b * a.region_bytes, &maps.in[b], 0, a.c0, a.amin[b] - a.amin_min, 0, slot_idx, fbar);
            if (a.shift_box_bytes && !dbg_noshift)
              tma_load_5d(dst + b * a.region_bytes + a.shift_off, &maps.in_shift[b], 0, a.c0 + 1,
                          a.amin[b] - a.amin_min, 0, slot_idx, fbar);
          } else if (a.planes_e2) {  // core-column planes: {folded-col run, row, plane, image}
            tma_load_4d(dst + b * a.region_bytes, &maps.in[b], a.c0 * a.planes_e2, oh0 + a.amin[b], 0, n, fbar);
            if (a.shift_box_bytes && !dbg_noshift)
              tma_load_4d(dst + b * a.region_bytes + a.shift_off, &maps.in_shift[b], (a.c0 + 1) * a.planes_e2,
                          oh0 + a.amin[b], 0, n, fbar);
          } else {
            tma_load_5d(dst + b * a.region_bytes, &maps.in[b], 0, a.c0, oh0 + a.amin[b], 0, n, fbar);
            if (a.shift_box_bytes && !dbg_noshift)
              tma_load_5d(dst + b * a.region_bytes + a.shift_off, &maps.in_shift[b], 0, a.c0 + 1, oh0 + a.amin[b], 0,
                          n, fbar);
          }
        }
      }
#if WFB_PROFILE
      if (pdbg)
        printf("tma producer cta0: %d units, %lld cycles: wait ring slot %lld, wait free A stage %lld\n", it,
               clock64() - p_all, p_ring, p_stage);
#endif
      if constexpr (kMc) {
        // producer tail: wait for the final release of every stage in use --
        // the peer's last multicast commit lands on this CTA's empty
        // barriers -- so no remote arrive is in flight at teardown
        for (int i = max(0, it - a.stages); i < it; ++i)
          mbar_wait(bar_empty + 8 * (i % a.stages), static_cast<uint32_t>(i / a.stages) & 1u);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    // The whole warp walks the (warp-uniform) schedule so descriptors live in
    // uniform registers straight from the constant bank; one lane issues.
    const bool skip_mma = prof(a, 0x100);  // profiling switch
    const bool no_wait = prof(a, 0x200000);  // profiling: issue the schedule back to back (with 0x1200)
    // descriptor start fields are 14-bit CTA-local offsets (>> 4): in a
    // cluster launch a rank-1 CTA's shared::cta addresses carry 0x1000000,
    // which must not spill into the LBO field
    const uint32_t b_lo = ((base + a.off_b) & 0x3FFFFu) >> 4;
    const uint32_t a_hi = a.a_desc_hi;
    const bool leader = elect_one() && rank == 0;  // pair: the leader CTA issues for both SMs
    if (kPair == 2 && rank != 0) goto mma_done;
    mbar_wait(bar_b, 0);
    if (leader) tl_mark(a, gbase, 4);  // B landed
    if constexpr (kPair == 2) mbar_wait_cluster(bar_bpeer, 0);
    {
    // Per-tile scalars read once (laundering them into registers with opq()
    // measured the same: the issuer's remaining gap to the tensor pipe is
    // elsewhere).
    const int ksplit = a.ksplit, tps = a.tps, stages = a.stages, stage_bytes = a.stage_bytes;
    const int tile_shift = a.tile_shift, n_acc = a.n_acc, acc_shift = a.acc_shift;
    const int num_units = a.num_units, unit_stride = a.unit_stride;
    const uint32_t acc_stride = a.acc_stride;
    const uint32_t a_base = base + a.off_a;
    const int nt_e0 = a.nt_entry0[ntile], nt_en = a.nt_entries[ntile], nt_sp = a.nt_split[ntile];
    // profiling (0x80000, CTA 0): cycles the issuer waits on the accumulator / the A stage
    const bool dbg = prof(a, 0x80000) && blockIdx.x == 0;
    long long w_acc = 0, w_full = 0, w_hi = 0, t_all = dbg ? clock64() : 0;
    unsigned long long ns_all = 0;  // wall time of the same span: cycles / ns = the SM clock it ran at
#if WFB_PROFILE
    if (dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns_all));
#endif
    int tile = 0;
    int ring_slot = 0;         // kProd 5: the unit's ring slot, freed once its A stage landed
    int stage_c = 0;           // A stage of the next sub-stage (kept incrementally: no division per tile)
    uint32_t round_c = 0;      // its fill round
    for (int u = local; u < num_units; u += unit_stride) {
     const int stage_u = stage_c;  // the unit's first sub-stage
     const uint32_t round_u = round_c;
     for (int k = 0; k < tps; ++k, ++tile) {  // tps M tiles share the unit's A stage
      const int acc = tile & (n_acc - 1);
      const uint32_t acc_round = static_cast<uint32_t>(tile >> acc_shift);
      const int split = (ksplit == 1) ? nt_sp : -1;
      long long t0 = dbg ? clock64() : 0;
      if (!no_wait) {
        mbar_wait(bar_tempty + 8 * acc, (acc_round & 1u) ^ 1u);
        if (split < 0) mbar_wait(bar_tempty_hi + 8 * acc, (acc_round & 1u) ^ 1u);
      }
      if (dbg) { const long long t1 = clock64(); w_acc += t1 - t0; t0 = t1; }
      const uint32_t d_base = tmem_base + acc * acc_stride;
      int stage = stage_u;
      uint32_t round = round_u;
      for (int ks = 0; ks < ksplit; ++ks) {
        if (ks > 0 && ++stage == stages) { stage = 0; ++round; }
        const int e0 = (ksplit == 1) ? nt_e0 : a.ks_entry0[ks];
        const int entries = (ksplit == 1) ? nt_en : a.ks_entries[ks];
        if (k == 0 && !no_wait) mbar_wait(bar_full + 8 * stage, round & 1u);
        if (leader && tile == 0 && ks == 0) tl_mark(a, gbase, 5);  // first A stage landed
        if constexpr (kProd == 5) {
          if (k == 0 && ks == 0 && leader) {
            if constexpr (kMc) {  // the shared slot is free once both CTAs' stages landed
              mbar_arrive_cluster(mapa(bar_raw_empty + 8 * ring_slot, 0));
              mbar_arrive_cluster(mapa(bar_raw_empty + 8 * ring_slot, 1));
            } else {
              mbar_arrive(bar_raw_empty + 8 * ring_slot);
            }
          }
        }
        if (dbg) { const long long t1 = clock64(); w_full += t1 - t0; t0 = t1; }
        tc_fence_after();
        const uint32_t a_lo = ((a_base + stage * stage_bytes + k * tile_shift) & 0x3FFFFu) >> 4;
        if (!skip_mma) {
          int i = 0;
          if (split > 0) {  // lower half first, then wait for the epilogue to drain the upper half
            for (; i < split; ++i) {
              const uint4 e = a.table[e0 + i];
              const uint64_t adesc = (static_cast<uint64_t>(a_hi) << 32) | (e.x + a_lo);
              const uint64_t bdesc = (static_cast<uint64_t>(0x4008u) << 32) | (e.y + b_lo);
              if (leader) issue_mma<kKind, kPair>(d_base + e.w, adesc, bdesc, e.z & 0x7FFFFFFFu, e.z >> 31);
            }
            if (dbg) t0 = clock64();
            if (!no_wait) mbar_wait(bar_tempty_hi + 8 * acc, (acc_round & 1u) ^ 1u);
            if (dbg) w_hi += clock64() - t0;
            tc_fence_after();
          }
          for (; i + kIssueGroup <= entries; i += kIssueGroup) {
#pragma unroll
            for (int j = 0; j < kIssueGroup; ++j) {
              const uint4 e = a.table[e0 + i + j];
              const uint64_t adesc = (static_cast<uint64_t>(a_hi) << 32) | (e.x + a_lo);
              const uint64_t bdesc = (static_cast<uint64_t>(0x4008u) << 32) | (e.y + b_lo);
              if (leader) issue_mma<kKind, kPair>(d_base + e.w, adesc, bdesc, e.z & 0x7FFFFFFFu, e.z >> 31);
            }
          }
          for (; i < entries; ++i) {
            const uint4 e = a.table[e0 + i];
            const uint64_t adesc = (static_cast<uint64_t>(a_hi) << 32) | (e.x + a_lo);
            const uint64_t bdesc = (static_cast<uint64_t>(0x4008u) << 32) | (e.y + b_lo);
            if (leader) issue_mma<kKind, kPair>(d_base + e.w, adesc, bdesc, e.z & 0x7FFFFFFFu, e.z >> 31);
          }
        }
        else if (split > 0) {
          mbar_wait(bar_tempty_hi + 8 * acc, (acc_round & 1u) ^ 1u);
        }
        if (leader && k == tps - 1) {  // last tile frees the stage (multicast: in both CTAs)
          if constexpr (kMc) {
            if (prof(a, 0x2000)) mma_commit(bar_empty + 8 * stage);
            else mma_commit_mc(bar_empty + 8 * stage, 0x3);
          }
          else commit_to<kPair>(bar_empty + 8 * stage);
        }
      }
      if (leader) commit_to<kPair>(bar_tfull + 8 * acc);
      if (leader) tl_mark(a, gbase, 6);  // last MMA of the tile issued
      __syncwarp();
     }
     for (int ks = 0; ks < ksplit; ++ks)  // advance past the unit's sub-stages
       if (++stage_c == stages) { stage_c = 0; ++round_c; }
     if constexpr (kProd == 5)
       if (++ring_slot == a.raw_slots) ring_slot = 0;
    }
#if WFB_PROFILE
    if (dbg && leader)
    {
      unsigned long long ns_end;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns_end));
      const long long cyc = clock64() - t_all;
      printf("mma issuer cta0: %d tiles, %lld cycles in %llu ns (%.0f MHz): wait accumulator %lld (upper half %lld), "
             "wait A stage %lld\n", tile, cyc, ns_end - ns_all, 1e3 * cyc / (double)(ns_end - ns_all), w_acc, w_hi, w_full);
    }
#endif
    }
  mma_done:;
  } else if (warp >= 2 && warp < 10) {
    // ===================== epilogue (warps 2..9) =====================
    // Warp w owns TMEM lanes [32q, 32q+32), q = w % 4, and every other
    // CH-column chunk (half = 0 for warps 2..5, 1 for warps 6..9). Per chunk
    // and 16-lane half: tcgen05.ld.16x256b -> +bias (registers) -> ReLU ->
    // convert -> one 32-byte store per row. The packed filter permuted the
    // accumulator columns (chunk_perm, plan.hpp) so thread t holds CH/4
    // consecutive output channels of rows t/4 and t/4+8: the 4 threads of a
    // row write whole 128-byte lines, 8 rows per store instruction.
    constexpr int VPT = CH / 4;    // consecutive output channels per thread and row
    constexpr int NREG = CH / 2;   // registers per 16x256b load (two rows)
    constexpr int CPW = 256 / CH;  // chunks per warp at the maximum N-tile width (256), ping-pong mode
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int nchunks = ncols / CH;
    // Two ways to share a tile among the 8 warps. Default: warps 2..5 take the
    // even chunks, 6..9 the odd ones, of every tile. Ping-pong (a.epi_pp):
    // warps 2..5 take every chunk of the even tiles, 6..9 of the odd ones, so
    // two tiles drain at once (per-tile latency overlaps when N is narrow).
    const bool pp = a.epi_pp != 0;
    const int c_first = pp ? 0 : half, c_step = pp ? 1 : 2;
    const int nc_w = pp ? nchunks : ((nchunks > half) ? (nchunks - half + 1) / 2 : 0);  // this warp's chunks
    const int n_it = 2 * nc_w;                                                            // x two 16-lane halves
    // accumulator half-split: iterations [0, lo_it) read the lower half of the columns
    const bool split_acc = a.nt_split[ntile] > 0 && a.ksplit == 1;
    const int lo_it = split_acc ? (pp ? 2 * (nchunks / 2) : 2 * ((nchunks / 2 - half + 1) / 2)) : n_it;
    const int k4 = lane & 3;
    const bool relu = (a.epi_flags & WF_EPI_RELU) != 0;
    const bool dbg_skip_epi = prof(a, 0x200);
    const bool dbg_skip_store = prof(a, 0x400);
    const bool skip_ld = prof(a, 0x800);
    const bool stream_st = prof(a, 0x100000);  // experiment: streaming store hints
    float* const sbias = reinterpret_cast<float*>(gbase + a.off_bias);
    {  // bias slice of this N-tile into shared memory (off the producer's critical path)
      const bool has_bias = (a.bias != nullptr) && (a.epi_flags & WF_EPI_BIAS);
      for (int i = threadIdx.x - 64; i < ncols; i += 256) sbias[i] = has_bias ? a.bias[col0 + i] : 0.0f;
      named_bar_sync(1, 256);  // the 8 epilogue warps
    }
    // chunk cc of this warp is accumulator chunk c_first + c_step * cc; its output
    // column comes from the slot order (chunk_col), read per iteration
    // the four M rows this thread stores: (16-lane half h16, row group r8).
    // Everything about them that does not depend on the tile is computed once:
    // output row t of the tile, byte offset from the tile's first output pixel,
    // tile-independent validity, and per chunk the OW % r tail mask.
    int row_t[2][2];
    long long row_off[2][2];
    bool row_ok[2][2];
    unsigned row_cc[2][2];  // bit cc: this row's channels of chunk cc exist (ow < OW)
#pragma unroll
    for (int h16 = 0; h16 < 2; ++h16)
#pragma unroll
      for (int r8 = 0; r8 < 2; ++r8) {
        const int m = quarter * 32 + h16 * 16 + r8 * 8 + (lane >> 2);
        const int t = m / a.Wbox, wq = m - t * a.Wbox;
        row_t[h16][r8] = t;
        row_off[h16][r8] = (static_cast<long long>(t) * a.OW + wq * a.r) * a.Cout * static_cast<long long>(sizeof(OutT));
        row_ok[h16][r8] = (wq < a.Wfo) && (t < a.OHt) && !dbg_skip_store;
        unsigned bits = 0;
        for (int cc = 0; cc < nc_w; ++cc) {
          const int jsub = (a.chunk_col[ntile][c_first + c_step * cc] + VPT * k4) / a.Cout;  // output sub-column j
          bits |= (wq * a.r + jsub < a.OW) ? (1u << cc) : 0u;
        }
        row_cc[h16][r8] = bits;
      }
    const long long img_bytes = static_cast<long long>(a.OH) * a.OW * a.Cout * static_cast<long long>(sizeof(OutT));
    const long long orow_bytes = static_cast<long long>(a.OW) * a.Cout * static_cast<long long>(sizeof(OutT));
    // (image, first output row) of the current stage unit, advanced without
    // divisions: v = u (two-tile stages, divisor = units per image) or the M
    // tile u*kPair + rank (one tile per stage, divisor = M tiles per image)
    const int vdiv = (a.tps > 1) ? a.uph : a.ohb;
    const int vstep = (a.tps > 1) ? a.unit_stride : a.unit_stride * kPair;
    const int vq = vstep / vdiv, vr = vstep - (vstep / vdiv) * vdiv;
    const int v0 = (a.tps > 1) ? local : local * kPair + static_cast<int>(rank);
    int vn = v0 / vdiv, vrem = v0 - (v0 / vdiv) * vdiv;
    int it_tile = 0;
    // pair: arrivals go to the leader's accumulator-free barriers
    const uint32_t te_lo = (kPair == 2) ? mapa(bar_tempty, 0) : bar_tempty;
    const uint32_t te_hi = (kPair == 2) ? mapa(bar_tempty_hi, 0) : bar_tempty_hi;
    // profiling (0x400000, with 0x200000): the epilogue warps sit the launch out
    for (int u = prof(a, 0x400000) ? a.num_units : local; u < a.num_units; u += a.unit_stride) {
     const int vn_u = vn, vrem_u = vrem;
     vn += vq;
     vrem += vr;
     if (vrem >= vdiv) { vrem -= vdiv; ++vn; }
     for (int k = 0; k < a.tps; ++k, ++it_tile) {  // tile k of stage unit u
      if (pp && (it_tile & 1) != half) continue;  // the other warp group drains this tile
      const int acc = it_tile & (a.n_acc - 1);
      const uint32_t acc_round = static_cast<uint32_t>(it_tile >> a.acc_shift);
      const int mt = u * kPair + static_cast<int>(rank);  // (im2col rows; tps == 1 there)
      const int n = vn_u;
      const int oh0 = (a.tps > 1) ? (vrem_u * a.tps + k) * a.OHt : vrem_u * a.OHt;
      mbar_wait(bar_tfull + 8 * acc, acc_round & 1u);
      if (warp == 2 && lane == 0 && it_tile == 0) tl_mark(a, gbase, 7);  // accumulator ready
      tc_fence_after();
      if (dbg_skip_epi || n_it == 0) {
        tc_fence_before();
        arrive_at<kPair>(te_lo + 8 * acc);
        arrive_at<kPair>(te_hi + 8 * acc);
        continue;
      }
      uint8_t* rowp[2][2];  // first output pixel of the row (its j = 0 sub-column)
      bool rowv[2][2];
      unsigned rowc[2][2];
      uint8_t* const tile_out = a.out + n * img_bytes + oh0 * orow_bytes;
#pragma unroll
      for (int h16 = 0; h16 < 2; ++h16)
#pragma unroll
        for (int r8 = 0; r8 < 2; ++r8) {
          if constexpr (kProd == 2) {  // im2col: M row = flattened output pixel, one per row
            const long long P = static_cast<long long>(mt) * 128 + quarter * 32 + h16 * 16 + r8 * 8 + (lane >> 2);
            rowv[h16][r8] = (P < a.total_px) && !dbg_skip_store;
            rowp[h16][r8] = a.out + P * a.row_bytes;
            rowc[h16][r8] = ~0u;
          } else {
            rowv[h16][r8] = row_ok[h16][r8] && (oh0 + row_t[h16][r8] < a.OH) && (n < a.n_img);
            rowp[h16][r8] = tile_out + row_off[h16][r8];
            rowc[h16][r8] = row_cc[h16][r8];
          }
        }
      const uint32_t tq = tmem_base + acc * a.acc_stride + (static_cast<uint32_t>(quarter * 32) << 16);
      // iteration it: chunk cc = it / 2 (c = half + 2cc), 16-lane half h16 = it % 2
      auto taddr = [&](int it) {
        return tq + (static_cast<uint32_t>((it & 1) * 16) << 16) +
               static_cast<uint32_t>((c_first + c_step * (it >> 1)) * CH);
      };
      if (lo_it == 0) arrive_at<kPair>(te_lo + 8 * acc);  // this warp reads no lower-half column
      uint32_t buf[2][NREG];
      tmem_ld_16x256b<NREG>(taddr(0), buf[0], skip_ld);
#pragma unroll
      for (int it = 0; it < 2 * CPW; ++it) {
        if (it >= n_it) break;
        tmem_ld_wait();
        reg_fence<NREG>(buf[it & 1]);
        if (it + 1 < n_it) tmem_ld_16x256b<NREG>(taddr(it + 1), buf[(it + 1) & 1], skip_ld);
        const int cc = it >> 1, h16 = it & 1;
        const uint32_t(&r)[NREG] = buf[it & 1];
        const int ocol = a.chunk_col[ntile][c_first + c_step * cc];  // slot order -> output column
        const long long coff = static_cast<long long>(ocol + VPT * k4) * sizeof(OutT);
        float bb[VPT];  // bias of this thread's VPT channels (16-byte shared loads; registers are tight)
#pragma unroll
        for (int q = 0; q < VPT / 4; ++q) {
          const float4 t4 = reinterpret_cast<const float4*>(sbias + ocol - col0 + VPT * k4)[q];
          bb[4 * q] = t4.x; bb[4 * q + 1] = t4.y; bb[4 * q + 2] = t4.z; bb[4 * q + 3] = t4.w;
        }
#pragma unroll
        for (int r8 = 0; r8 < 2; ++r8) {
          float v[VPT];
#pragma unroll
          for (int i = 0; i < CH / 8; ++i) {
            v[2 * i] = __uint_as_float(r[4 * i + 2 * r8]) + bb[2 * i];
            v[2 * i + 1] = __uint_as_float(r[4 * i + 2 * r8 + 1]) + bb[2 * i + 1];
          }
          if (relu) {
#pragma unroll
            for (int k = 0; k < VPT; ++k) v[k] = (v[k] < 0.0f) ? 0.0f : v[k];
          }
          if (rowv[h16][r8] && ((rowc[h16][r8] >> cc) & 1u)) {
            if (stream_st) store_row<OutT, VPT, true>(rowp[h16][r8] + coff, v);
            else store_row<OutT, VPT, false>(rowp[h16][r8] + coff, v);
          }
        }
        if (it + 1 == lo_it) {  // lower half of the accumulator read (its wait::ld is done)
          tc_fence_before();
          arrive_at<kPair>(te_lo + 8 * acc);
        }
      }
      tc_fence_before();
      arrive_at<kPair>(te_hi + 8 * acc);
     }
    }
  }

  if (warp == 2 && lane == 0) tl_mark(a, gbase, 8);  // epilogue warp 2 done (stores issued)
  tc_fence_before();
  // pair: the leader's MMAs wrote this CTA's TMEM; multicast: no CTA leaves
  // while the peer may still commit to its barriers
  if constexpr (kPair == 2 || kMc) cluster_sync();
  else __syncthreads();
#if WFB_PROFILE
  if ((a.epi_flags & 0x8000) && blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long* t = reinterpret_cast<const unsigned long long*>(gbase + 1536);
    unsigned long long te;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(te));
    printf("timeline cta0 (ns after entry): prologue %llu | B issued %llu | prev grid done %llu | B landed %llu | "
           "A landed %llu | last MMA issued %llu | acc ready %llu | epilogue done %llu | exit sync %llu\n",
           t[1] - t[0], t[2] - t[0], t[3] - t[0], t[4] - t[0], t[5] - t[0], t[6] - t[0], t[7] - t[0], t[8] - t[0],
           te - t[0]);
  }
#endif
  if (warp == 1) {
    tc_fence_after();
    if constexpr (kPair == 2) tmem_dealloc_pair(tmem_base, a.tmem_cols);
    else tmem_dealloc(tmem_base, a.tmem_cols);
  }
}

// Kernel selectors: the device function for one (producer, MMA kind, output
// type, epilogue chunk[, pair | multicast]) combination, or nullptr when the
// combination is not built. Instantiated in conv_prod<kProd>.cu / conv_pair.cu;
// conv_fold.cu launches them with cudaLaunchKernelExC.
template <int kKind, typename OutT, int CH, int kProd, int kPair = 1, int kMc = 0>
const void* kernel_ptr() {
  return reinterpret_cast<const void*>(&conv_fold_kernel<kKind, OutT, CH, kProd, kPair, kMc>);
}

// kind: 0 kind::f16, 1 kind::tf32; out: output dtype; ch: epilogue chunk.
template <int kProd>
const void* conv_kernel_fn(int kind, wf_dtype out, int ch) {
  if constexpr (kProd == 4 || kProd == 5) {  // kind::f16, 32-column chunks (576 threads: CH=64 would spill)
    if (kind == 1 || ch != 32) return nullptr;
    if (out == WF_BF16) return kernel_ptr<0, __nv_bfloat16, 32, kProd>();
    if (out == WF_F16) return kernel_ptr<0, __half, 32, kProd>();
    return kernel_ptr<0, float, 32, kProd>();
  } else {
    if constexpr (kProd != 0) {
      if (kind == 1) return nullptr;  // tf32 runs with the TMA producer only
    } else if (kind == 1) {
      if (ch != 32) return nullptr;
      if (out == WF_BF16) return kernel_ptr<1, __nv_bfloat16, 32, kProd>();
      if (out == WF_F16) return kernel_ptr<1, __half, 32, kProd>();
      return kernel_ptr<1, float, 32, kProd>();
    }
    if (ch == 64) {
      if (out == WF_BF16) return kernel_ptr<0, __nv_bfloat16, 64, kProd>();
      if (out == WF_F16) return kernel_ptr<0, __half, 64, kProd>();
      return kernel_ptr<0, float, 64, kProd>();
    }
    if (out == WF_BF16) return kernel_ptr<0, __nv_bfloat16, 32, kProd>();
    if (out == WF_F16) return kernel_ptr<0, __half, 32, kProd>();
    return kernel_ptr<0, float, 32, kProd>();
  }
}

// CTA-pair kernel (cluster of 2, cta_group::2 MMAs), TMA producer, kind::f16.
const void* conv_kernel_fn_pair(wf_dtype out, int ch);
// 2-CTA N-tile cluster with multicast A loads, TMA producer, kind::f16.
const void* conv_kernel_fn_mc(wf_dtype out, int ch);
// the same cluster fed by the in-kernel L2 ring (kProd 5), 32-column chunks
const void* conv_kernel_fn_mc5(wf_dtype out);

extern template const void* conv_kernel_fn<0>(int, wf_dtype, int);
extern template const void* conv_kernel_fn<1>(int, wf_dtype, int);
extern template const void* conv_kernel_fn<2>(int, wf_dtype, int);
extern template const void* conv_kernel_fn<4>(int, wf_dtype, int);
extern template const void* conv_kernel_fn<5>(int, wf_dtype, int);

}  // namespace wfb
