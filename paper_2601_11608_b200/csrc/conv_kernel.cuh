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
//                kProd 1/2: with warps 10..11, a software gather (16-byte
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

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "kernels.hpp"
#include "ptx.cuh"

namespace wfb {

constexpr int kMaxTable = 384;  // schedule entries per launch (constant bank)
constexpr int kGatherWarps = 3;  // software-gather producer: warp 0 + warps 10, 11
constexpr int kMaxKsplit = 8;    // A stages per M tile (im2col kh ranges)

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
  int nt_bbytes[kMaxNTiles];
  long long nt_bsrc[kMaxNTiles];  // device address of the N-tile's packed B
  long long row_bytes;            // bytes of one folded output row = r*Cout*out_elem
  int chunk_col[kMaxNTiles][kMaxAccCols / 32];  // output column of each epilogue chunk
  unsigned acc_stride, tmem_cols;
  int epi_flags;
  int off_a, off_b, off_bias;
  // software-gather producer (kProd 1: folded layout, 2: explicit im2col)
  const uint8_t* x;               // input base (16-byte aligned)
  long long in_row_bytes;         // W*C*elem (any alignment: AlexNet 1362 B)
  long long in_img_bytes;         // H*W*C*elem
  long long pix_bytes;            // folded pixel f*C*elem
  int H, Q, Qr, NR;               // core cols per pixel, regions per residue (+shift), rows per region
  int lbo_a;                      // bytes between core-column regions
  int n_gather_chunks;            // 16-byte chunks per A stage
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

// VPT consecutive output channels of one row -> global, 32-byte stores.
template <typename OutT, int VPT>
__device__ __forceinline__ void store_row(uint8_t* dst, const float (&v)[VPT]) {
  if constexpr (sizeof(OutT) == 4) {
    static_assert(VPT % 8 == 0, "fp32 rows are stored 8 values at a time");
#pragma unroll
    for (int q = 0; q < VPT / 8; ++q) {
      uint32_t pk[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) pk[k] = __float_as_uint(v[8 * q + k]);
      ptx::st_global_v8(dst + 32 * q, pk);
    }
  } else if constexpr (VPT == 16) {
    uint32_t pk[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) pk[k] = pack2<OutT>(v[2 * k], v[2 * k + 1]);
    ptx::st_global_v8(dst, pk);
  } else {
    static_assert(VPT == 8, "2-byte rows are 8 or 16 values");
    ptx::st_global_v4(dst, make_uint4(pack2<OutT>(v[0], v[1]), pack2<OutT>(v[2], v[3]), pack2<OutT>(v[4], v[5]),
                                      pack2<OutT>(v[6], v[7])));
  }
}

// Bytes [boff, boff+16) of an input row (any 2-byte alignment), bytes outside
// [0, rb) read as zero (the conv padding). Loads only the 16-byte aligned
// blocks that intersect the row.
__device__ __forceinline__ uint4 load16_row(const uint8_t* row, long long boff, long long rb) {
  if (boff >= rb || boff + 16 <= 0) return make_uint4(0u, 0u, 0u, 0u);
  const uintptr_t addr = reinterpret_cast<uintptr_t>(row) + boff;
  const uint32_t sh = static_cast<uint32_t>(addr & 15u);
  const long long b0 = boff - sh;  // row offset of the first aligned block
  const uint4 z = make_uint4(0u, 0u, 0u, 0u);
  const uint4 v0 = (b0 < rb && b0 + 16 > 0) ? __ldg(reinterpret_cast<const uint4*>(addr - sh)) : z;
  uint32_t w0 = v0.x, w1 = v0.y, w2 = v0.z, w3 = v0.w;
  if (sh != 0) {
    const uint4 v1 = (b0 + 16 < rb) ? __ldg(reinterpret_cast<const uint4*>(addr - sh + 16)) : z;
    uint32_t w4 = v1.x, w5 = v1.y, w6 = v1.z, w7 = v1.w;
    if (sh & 8) { w0 = w2; w1 = w3; w2 = w4; w3 = w5; w4 = w6; w5 = w7; }
    if (sh & 4) { w0 = w1; w1 = w2; w2 = w3; w3 = w4; w4 = w5; }
    if (sh & 2) {
      w0 = __funnelshift_r(w0, w1, 16); w1 = __funnelshift_r(w1, w2, 16);
      w2 = __funnelshift_r(w2, w3, 16); w3 = __funnelshift_r(w3, w4, 16);
    }
    if (sh & 1) {  // byte-aligned rows only occur with 1-byte elements (not used)
      w0 = __funnelshift_r(w0, w1, 8); w1 = __funnelshift_r(w1, w2, 8);
      w2 = __funnelshift_r(w2, w3, 8); w3 = __funnelshift_r(w3, w4, 8);
    }
  }
  if (boff < 0 || boff + 16 > rb) {  // row edge: zero the bytes outside [0, rb)
    uint32_t w[4] = {w0, w1, w2, w3};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t m = 0;
#pragma unroll
      for (int bb = 0; bb < 4; ++bb) {
        const long long o = boff + 4 * k + bb;
        if (o >= 0 && o < rb) m |= 0xFFu << (8 * bb);
      }
      w[k] &= m;
    }
    w0 = w[0]; w1 = w[1]; w2 = w[2]; w3 = w[3];
  }
  return make_uint4(w0, w1, w2, w3);
}

// One A stage built by the gather warps: chunk d (16 bytes) of the stage.
template <int kProd>
__device__ __forceinline__ void gather_chunk(const ConvArgs& a, int d, int mt, int kh0, uint32_t& dst_off, uint4& v) {
  if constexpr (kProd == 1) {
    // folded layout, identical to the TMA boxes: [residue b][region q'][row i][folded col w''][16 B]
    const int w2 = d % a.Wbox;
    int t = d / a.Wbox;
    const int i = t % a.NR;
    t /= a.NR;
    const int qq = t % a.Qr;
    const int b = t / a.Qr;
    dst_off = static_cast<uint32_t>(b * a.region_bytes + qq * a.lbo_a + (i * a.Wbox + w2) * 16);
    const int n = mt / a.ohb;
    const int oh0 = (mt - n * a.ohb) * a.OHt;
    const int ih = (oh0 + a.amin[b] + i) * a.s + b;
    if (!((a.res_mask >> b) & 1u) || ih < 0 || ih >= a.H) {
      v = make_uint4(0u, 0u, 0u, 0u);
      return;
    }
    const int shift = (qq == a.Q) ? 1 : 0;
    const long long boff = static_cast<long long>(a.c0 + w2 + shift) * a.pix_bytes + (shift ? 0 : qq) * 16;
    v = load16_row(a.x + n * a.in_img_bytes + ih * a.in_row_bytes, boff, a.in_row_bytes);
  } else {
    // explicit im2col: [kh*U + u][core col cc][M row m][16 B]; row m = output pixel mt*128 + m
    const int m = d & 127;
    const int t = d >> 7;
    const int cc = t & 1;
    const int rg = t >> 1;
    const int khl = rg / a.U;  // kh relative to the sub-stage
    const int u = rg - khl * a.U;
    const int kh = kh0 + khl;
    dst_off = static_cast<uint32_t>(rg * 4096 + cc * 2048 + m * 16);
    const long long P = static_cast<long long>(mt) * 128 + m;
    if (P >= a.total_px) {
      v = make_uint4(0u, 0u, 0u, 0u);
      return;
    }
    const long long per_img = static_cast<long long>(a.OH) * a.OW;
    const int n = static_cast<int>(P / per_img);
    const int rem = static_cast<int>(P - n * per_img);
    const int oh = rem / a.OW;
    const int ow = rem - oh * a.OW;
    const int ih = oh * a.s - a.ph + kh;
    if (ih < 0 || ih >= a.H) {
      v = make_uint4(0u, 0u, 0u, 0u);
      return;
    }
    const long long boff = static_cast<long long>(ow * a.sw - a.pw) * a.pix_bytes + (2 * u + cc) * 16;
    v = load16_row(a.x + n * a.in_img_bytes + ih * a.in_row_bytes, boff, a.in_row_bytes);
  }
}

template <int kKind, typename OutT, int CH, int kProd>
__global__ void __launch_bounds__(kProd == 0 ? 320 : 384, 1)
    conv_fold_kernel(const __grid_constant__ ConvArgs a, const __grid_constant__ TmaMaps maps) {
  using namespace ptx;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t bar_full = base;          // [stages] x 8 B
  const uint32_t bar_empty = base + 64;    // [stages] x 8 B
  const uint32_t bar_tfull = base + 128;   // [2] x 8 B
  const uint32_t bar_tempty = base + 144;  // [2] x 8 B
  const uint32_t bar_b = base + 160;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + 192);

  // warp index via shuffle so the compiler knows it is warp-uniform (keeps the
  // MMA issuer's operands in uniform registers)
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const int ntile = blockIdx.x % a.n_tiles;
  const int local = blockIdx.x / a.n_tiles;
  const int ncols = a.nt_cols[ntile];
  const int col0 = a.nt_col0[ntile];

  {  // bias slice of this N-tile into shared memory
    float* sbias = reinterpret_cast<float*>(gbase + a.off_bias);
    const bool has_bias = (a.bias != nullptr) && (a.epi_flags & WF_EPI_BIAS);
    for (int i = threadIdx.x; i < ncols; i += blockDim.x) sbias[i] = has_bias ? a.bias[col0 + i] : 0.0f;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < a.stages; ++i) {
      mbar_init(bar_full + 8 * i, kProd == 0 ? 1 : kGatherWarps);  // TMA: one expect_tx; gather: one arrive per warp
      mbar_init(bar_empty + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar_tfull + 8 * i, 1);
      mbar_init(bar_tempty + 8 * i, 256);
    }
    mbar_init(bar_b, 1);
    fence_barrier_init();
  }
  if (kProd == 0 && warp == 0 && lane == 0) {
    for (int b = 0; b < a.s; ++b)
      if ((a.res_mask >> b) & 1u) {
        prefetch_tmap(&maps.in[b]);
        if (a.shift_box_bytes) prefetch_tmap(&maps.in_shift[b]);
      }
  }
  if (warp == 1) tmem_alloc(smem_u32(tmem_slot), a.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (kProd != 0 && (warp == 0 || warp >= 10)) {
    // ===================== gather producer (warps 0, 10, 11) =====================
    // Builds each A stage with 16-byte global loads (any row alignment,
    // zero-filled padding) and st.shared; rows of AlexNet's 1362-byte pitch
    // and the explicit im2col of the unfolded variant cannot be TMA boxes.
    if (warp == 0 && elect_one()) {
      const uint8_t* gb = reinterpret_cast<const uint8_t*>(a.nt_bsrc[ntile]);
      const int bb = a.nt_bbytes[ntile];
      mbar_arrive_expect_tx(bar_b, static_cast<uint32_t>(bb));
      for (int off = 0; off < bb; off += 32768)
        bulk_g2s(base + a.off_b + off, gb + off, static_cast<uint32_t>(min(32768, bb - off)), bar_b);
    }
    __syncwarp();
    constexpr int NGT = kGatherWarps * 32;
    const int gt = (warp == 0 ? 0 : warp - 9) * 32 + lane;  // 0..NGT-1
    int it = 0;
    for (int mt = local; mt < a.num_mtiles; mt += a.ctas_per_ntile) {
      for (int ks = 0; ks < a.ksplit; ++ks, ++it) {  // im2col: kh ranges of one M tile
        const int stage = it % a.stages;
        const uint32_t round = static_cast<uint32_t>(it / a.stages);
        mbar_wait(bar_empty + 8 * stage, (round & 1u) ^ 1u);
        const uint32_t dst = base + a.off_a + stage * a.stage_bytes;
        const int nch = (a.ksplit == 1) ? a.n_gather_chunks : a.ks_chunks[ks];
        const int kh0 = (a.ksplit == 1) ? 0 : a.ks_kh0[ks];
        if (!(a.epi_flags & 0x1000)) {
          int d = gt;
          for (; d + 3 * NGT < nch; d += 4 * NGT) {  // 4 loads in flight per thread
            uint32_t o[4];
            uint4 v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) gather_chunk<kProd>(a, d + k * NGT, mt, kh0, o[k], v[k]);
#pragma unroll
            for (int k = 0; k < 4; ++k) st_shared_v4(dst + o[k], v[k].x, v[k].y, v[k].z, v[k].w);
          }
          for (; d < nch; d += NGT) {
            uint32_t o;
            uint4 v;
            gather_chunk<kProd>(a, d, mt, kh0, o, v);
            st_shared_v4(dst + o, v.x, v.y, v.z, v.w);
          }
        }
        fence_proxy_async_smem();  // generic-proxy stores -> visible to tcgen05 (async proxy)
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_full + 8 * stage);
      }
    }
  } else if (warp == 0) {
    // ===================== TMA producer (one elected lane) =====================
    if (elect_one()) {
      const uint8_t* gb = reinterpret_cast<const uint8_t*>(a.nt_bsrc[ntile]);
      const int bb = a.nt_bbytes[ntile];
      mbar_arrive_expect_tx(bar_b, static_cast<uint32_t>(bb));
      for (int off = 0; off < bb; off += 32768)
        bulk_g2s(base + a.off_b + off, gb + off, static_cast<uint32_t>(min(32768, bb - off)), bar_b);
      const uint32_t tx = static_cast<uint32_t>((a.box_bytes + a.shift_box_bytes) * __popc(a.res_mask));
      int it = 0;
      for (int mt = local; mt < a.num_mtiles; mt += a.ctas_per_ntile, ++it) {
        const int stage = it % a.stages;
        const uint32_t round = static_cast<uint32_t>(it / a.stages);
        mbar_wait(bar_empty + 8 * stage, (round & 1u) ^ 1u);
        const int n = mt / a.ohb;
        const int oh0 = (mt - n * a.ohb) * a.OHt;
        const uint32_t dst = base + a.off_a + stage * a.stage_bytes;
        if (a.epi_flags & 0x1000) {  // profiling: no A loads (stage contents stale)
          mbar_arrive(bar_full + 8 * stage);
          continue;
        }
        mbar_arrive_expect_tx(bar_full + 8 * stage, tx);
        for (int b = 0; b < a.s; ++b) {
          if (!((a.res_mask >> b) & 1u)) continue;
          tma_load_5d(dst + b * a.region_bytes, &maps.in[b], 0, a.c0, oh0 + a.amin[b], 0, n, bar_full + 8 * stage);
          if (a.shift_box_bytes)
            tma_load_5d(dst + b * a.region_bytes + a.shift_off, &maps.in_shift[b], 0, a.c0 + 1, oh0 + a.amin[b], 0, n,
                        bar_full + 8 * stage);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    // The whole warp walks the (warp-uniform) schedule so descriptors live in
    // uniform registers straight from the constant bank; one lane issues.
    const bool skip_mma = (a.epi_flags & 0x100) != 0;  // profiling switch
    const uint32_t b_lo = (base + a.off_b) >> 4;
    const bool leader = elect_one();
    mbar_wait(bar_b, 0);
    int it = 0;  // A stages consumed (ksplit per M tile)
    int tile = 0;
    for (int mt = local; mt < a.num_mtiles; mt += a.ctas_per_ntile, ++tile) {
      const int acc = tile & 1;
      const uint32_t acc_round = static_cast<uint32_t>(tile >> 1);
      mbar_wait(bar_tempty + 8 * acc, (acc_round & 1u) ^ 1u);
      const uint32_t d_base = tmem_base + acc * a.acc_stride;
      for (int ks = 0; ks < a.ksplit; ++ks, ++it) {
        const int stage = it % a.stages;
        const uint32_t round = static_cast<uint32_t>(it / a.stages);
        const int e0 = (a.ksplit == 1) ? a.nt_entry0[ntile] : a.ks_entry0[ks];
        const int entries = (a.ksplit == 1) ? a.nt_entries[ntile] : a.ks_entries[ks];
        mbar_wait(bar_full + 8 * stage, round & 1u);
        tc_fence_after();
        const uint32_t a_lo = (base + a.off_a + stage * a.stage_bytes) >> 4;
        if (!skip_mma) {
          int i = 0;
          for (; i + 8 <= entries; i += 8) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const uint4 e = a.table[e0 + i + j];
              const uint64_t adesc = (static_cast<uint64_t>(0x4008u) << 32) | (e.x + a_lo);
              const uint64_t bdesc = (static_cast<uint64_t>(0x4008u) << 32) | (e.y + b_lo);
              if (leader) mma<kKind>(d_base + e.w, adesc, bdesc, e.z & 0x7FFFFFFFu, e.z >> 31);
            }
          }
          for (; i < entries; ++i) {
            const uint4 e = a.table[e0 + i];
            const uint64_t adesc = (static_cast<uint64_t>(0x4008u) << 32) | (e.x + a_lo);
            const uint64_t bdesc = (static_cast<uint64_t>(0x4008u) << 32) | (e.y + b_lo);
            if (leader) mma<kKind>(d_base + e.w, adesc, bdesc, e.z & 0x7FFFFFFFu, e.z >> 31);
          }
        }
        if (leader) mma_commit(bar_empty + 8 * stage);
      }
      if (leader) mma_commit(bar_tfull + 8 * acc);
      __syncwarp();
    }
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
    constexpr int CPW = 128 / CH;  // chunks per warp at the maximum N-tile width (256)
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int nchunks = ncols / CH;
    const int nc_w = (nchunks > half) ? (nchunks - half + 1) / 2 : 0;  // this warp's chunks
    const int n_it = 2 * nc_w;                                          // x two 16-lane halves
    const int k4 = lane & 3;
    const bool relu = (a.epi_flags & WF_EPI_RELU) != 0;
    const bool dbg_skip_epi = (a.epi_flags & 0x200) != 0;
    const bool dbg_skip_store = (a.epi_flags & 0x400) != 0;
    const bool skip_ld = (a.epi_flags & 0x800) != 0;
    const float* sbias = reinterpret_cast<const float*>(gbase + a.off_bias);
    float breg[CPW][VPT];   // bias of this thread's channels in each of its chunks
    long long coff[CPW];    // byte offset of each chunk's first output column in a row
    int jsub[CPW];          // output sub-column j of this thread's channels (OW % r tail mask)
#pragma unroll
    for (int cc = 0; cc < CPW; ++cc) {
      const int c = half + 2 * cc;
      const int ocol = (c < nchunks) ? a.chunk_col[ntile][c] : col0;  // slot order -> output column
      coff[cc] = static_cast<long long>(ocol + VPT * k4) * sizeof(OutT);
      jsub[cc] = (ocol + VPT * k4) / a.Cout;
#pragma unroll
      for (int v = 0; v < VPT; ++v) breg[cc][v] = (c < nchunks) ? sbias[ocol - col0 + VPT * k4 + v] : 0.0f;
    }
    // the four M rows this thread stores: (16-lane half h16, row group r8)
    int row_t[2][2], row_w[2][2];
#pragma unroll
    for (int h16 = 0; h16 < 2; ++h16)
#pragma unroll
      for (int r8 = 0; r8 < 2; ++r8) {
        const int m = quarter * 32 + h16 * 16 + r8 * 8 + (lane >> 2);
        row_t[h16][r8] = m / a.Wbox;
        row_w[h16][r8] = m - row_t[h16][r8] * a.Wbox;
      }
    int it_tile = 0;
    for (int mt = local; mt < a.num_mtiles; mt += a.ctas_per_ntile, ++it_tile) {
      const int acc = it_tile & 1;
      const uint32_t acc_round = static_cast<uint32_t>(it_tile >> 1);
      const int n = mt / a.ohb;
      const int oh0 = (mt - n * a.ohb) * a.OHt;
      mbar_wait(bar_tfull + 8 * acc, acc_round & 1u);
      tc_fence_after();
      if (dbg_skip_epi || n_it == 0) {
        tc_fence_before();
        mbar_arrive(bar_tempty + 8 * acc);
        continue;
      }
      uint8_t* rowp[2][2];  // first output pixel of the row (its j = 0 sub-column)
      bool rowv[2][2];
      int roww[2][2];       // first output column ow of the row
#pragma unroll
      for (int h16 = 0; h16 < 2; ++h16)
#pragma unroll
        for (int r8 = 0; r8 < 2; ++r8) {
          if constexpr (kProd == 2) {  // im2col: M row = flattened output pixel, one per row
            const long long P = static_cast<long long>(mt) * 128 + quarter * 32 + h16 * 16 + r8 * 8 + (lane >> 2);
            rowv[h16][r8] = (P < a.total_px) && !dbg_skip_store;
            rowp[h16][r8] = a.out + P * a.row_bytes;
            roww[h16][r8] = 0;
          } else {
            const int t = row_t[h16][r8], wq = row_w[h16][r8];
            const int oh = oh0 + t;
            rowv[h16][r8] = (wq < a.Wfo) && (t < a.OHt) && (oh < a.OH) && !dbg_skip_store;
            roww[h16][r8] = wq * a.r;
            rowp[h16][r8] = a.out + ((static_cast<long long>(n) * a.OH + oh) * a.OW + wq * a.r) * a.Cout *
                                        static_cast<long long>(sizeof(OutT));
          }
        }
      const uint32_t tq = tmem_base + acc * a.acc_stride + (static_cast<uint32_t>(quarter * 32) << 16);
      // iteration it: chunk cc = it / 2 (c = half + 2cc), 16-lane half h16 = it % 2
      auto taddr = [&](int it) {
        return tq + (static_cast<uint32_t>((it & 1) * 16) << 16) + static_cast<uint32_t>((half + 2 * (it >> 1)) * CH);
      };
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
#pragma unroll
        for (int r8 = 0; r8 < 2; ++r8) {
          float v[VPT];
#pragma unroll
          for (int i = 0; i < CH / 8; ++i) {
            v[2 * i] = __uint_as_float(r[4 * i + 2 * r8]) + breg[cc][2 * i];
            v[2 * i + 1] = __uint_as_float(r[4 * i + 2 * r8 + 1]) + breg[cc][2 * i + 1];
          }
          if (relu) {
#pragma unroll
            for (int k = 0; k < VPT; ++k) v[k] = (v[k] < 0.0f) ? 0.0f : v[k];
          }
          if (rowv[h16][r8] && roww[h16][r8] + jsub[cc] < a.OW) store_row<OutT, VPT>(rowp[h16][r8] + coff[cc], v);
        }
      }
      tc_fence_before();
      mbar_arrive(bar_tempty + 8 * acc);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, a.tmem_cols);
  }
}

// Typed launch for one producer kind (instantiated in conv_prod<kProd>.cu).
template <int kKind, typename OutT, int CH, int kProd>
cudaError_t launch_typed(const ConvArgs& args, const TmaMaps& maps, int grid, int smem, cudaStream_t st) {
  auto kern = conv_fold_kernel<kKind, OutT, CH, kProd>;
  static int configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  kern<<<grid, kProd == 0 ? 320 : 384, smem, st>>>(args, maps);
  return cudaGetLastError();
}

// kind: 0 kind::f16, 1 kind::tf32; out: output dtype; ch: epilogue chunk.
template <int kProd>
cudaError_t launch_conv_prod(const ConvArgs& args, const TmaMaps& maps, int grid, int smem, cudaStream_t st, int kind,
                             wf_dtype out, int ch) {
  if constexpr (kProd != 0) {
    if (kind == 1) return cudaErrorInvalidValue;  // tf32 runs with the TMA producer only
  } else if (kind == 1) {
    if (ch != 32) return cudaErrorInvalidValue;
    if (out == WF_BF16) return launch_typed<1, __nv_bfloat16, 32, kProd>(args, maps, grid, smem, st);
    if (out == WF_F16) return launch_typed<1, __half, 32, kProd>(args, maps, grid, smem, st);
    return launch_typed<1, float, 32, kProd>(args, maps, grid, smem, st);
  }
  if (ch == 64) {
    if (out == WF_BF16) return launch_typed<0, __nv_bfloat16, 64, kProd>(args, maps, grid, smem, st);
    if (out == WF_F16) return launch_typed<0, __half, 64, kProd>(args, maps, grid, smem, st);
    return launch_typed<0, float, 64, kProd>(args, maps, grid, smem, st);
  }
  if (out == WF_BF16) return launch_typed<0, __nv_bfloat16, 32, kProd>(args, maps, grid, smem, st);
  if (out == WF_F16) return launch_typed<0, __half, 32, kProd>(args, maps, grid, smem, st);
  return launch_typed<0, float, 32, kProd>(args, maps, grid, smem, st);
}

extern template cudaError_t launch_conv_prod<0>(const ConvArgs&, const TmaMaps&, int, int, cudaStream_t, int, wf_dtype,
                                                int);
extern template cudaError_t launch_conv_prod<1>(const ConvArgs&, const TmaMaps&, int, int, cudaStream_t, int, wf_dtype,
                                                int);
extern template cudaError_t launch_conv_prod<2>(const ConvArgs&, const TmaMaps&, int, int, cudaStream_t, int, wf_dtype,
                                                int);

}  // namespace wfb
