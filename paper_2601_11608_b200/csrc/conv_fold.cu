// conv_fold.cu -- K2: folded implicit-GEMM first-layer convolution for sm_100a.
//
// Replaces the reference hot loop widthfold::conv2d (src/refconv.cpp:57-78)
// run on the width-folded view (src/fold.cpp:113-143, a reshape) followed by
// bias_add (src/refconv.cpp:82-95) and reconstruct_output (src/fold.cpp:228-259,
// a reshape). One persistent, warp-specialised CTA per SM:
//
//   warp 0      TMA producer: once, the CTA's packed B operand (bulk copy);
//               per 128-row M tile, one 5-D TMA box per H-stride residue that
//               lands the canonical K-major core-matrix layout directly
//               (plan.hpp explains the view); OOB rows/cols are zero-filled,
//               which implements the conv padding.
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer, driven by the
//               schedule table (a_off, b_off, tmem column, accumulate) built by
//               plan.cpp; fp32 accumulators double-buffered in TMEM.
//   warps 2..5  epilogue: tcgen05.ld -> +bias -> ReLU -> bf16/fp16/fp32 ->
//               64B-swizzled staging smem -> TMA tensor store of final NHWC.
//
// Work split: CTA c serves N-tile (c % n_tiles) and M tiles
// local, local + ctas_per_ntile, ... -- the B operand of its N-tile stays
// resident in shared memory for the whole launch.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "kernels.hpp"
#include "ptx.cuh"

namespace wfb {

constexpr int kMaxTable = 384;  // schedule entries per launch (constant bank)

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

template <int kKind, typename OutT, int CH>
__global__ void __launch_bounds__(320, 1)
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
      mbar_init(bar_full + 8 * i, 1);
      mbar_init(bar_empty + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar_tfull + 8 * i, 1);
      mbar_init(bar_tempty + 8 * i, 256);
    }
    mbar_init(bar_b, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
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

  if (warp == 0) {
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
    const int e0 = a.nt_entry0[ntile];
    const int entries = a.nt_entries[ntile];
    const bool skip_mma = (a.epi_flags & 0x100) != 0;  // profiling switch
    const uint32_t b_lo = (base + a.off_b) >> 4;
    const bool leader = elect_one();
    mbar_wait(bar_b, 0);
    int it = 0;
    for (int mt = local; mt < a.num_mtiles; mt += a.ctas_per_ntile, ++it) {
      const int stage = it % a.stages;
      const uint32_t round = static_cast<uint32_t>(it / a.stages);
      const int acc = it & 1;
      const uint32_t acc_round = static_cast<uint32_t>(it >> 1);
      mbar_wait(bar_tempty + 8 * acc, (acc_round & 1u) ^ 1u);
      mbar_wait(bar_full + 8 * stage, round & 1u);
      tc_fence_after();
      const uint32_t a_lo = (base + a.off_a + stage * a.stage_bytes) >> 4;
      const uint32_t d_base = tmem_base + acc * a.acc_stride;
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
      if (leader) {
        mma_commit(bar_empty + 8 * stage);
        mma_commit(bar_tfull + 8 * acc);
      }
      __syncwarp();
    }
  } else {
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
#pragma unroll
    for (int cc = 0; cc < CPW; ++cc) {
      const int c = half + 2 * cc;
      const int ocol = (c < nchunks) ? a.chunk_col[ntile][c] : col0;  // slot order -> output column
      coff[cc] = static_cast<long long>(ocol) * sizeof(OutT);
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
    const long long col_bytes = static_cast<long long>(VPT * k4) * sizeof(OutT);
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
      uint8_t* rowp[2][2];
      bool rowv[2][2];
#pragma unroll
      for (int h16 = 0; h16 < 2; ++h16)
#pragma unroll
        for (int r8 = 0; r8 < 2; ++r8) {
          const int t = row_t[h16][r8], wq = row_w[h16][r8];
          const int oh = oh0 + t;
          rowv[h16][r8] = (wq < a.Wfo) && (t < a.OHt) && (oh < a.OH) && !dbg_skip_store;
          rowp[h16][r8] = a.out + ((static_cast<long long>(n) * a.OH + oh) * a.Wfo + wq) * a.row_bytes + col_bytes;
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
          if (rowv[h16][r8]) store_row<OutT, VPT>(rowp[h16][r8] + coff[cc], v);
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

template <int kKind, typename OutT, int CH>
cudaError_t launch_typed(const ConvArgs& args, const TmaMaps& maps, int grid, int smem, cudaStream_t st) {
  auto kern = conv_fold_kernel<kKind, OutT, CH>;
  static int configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  kern<<<grid, 320, smem, st>>>(args, maps);
  return cudaGetLastError();
}

}  // namespace

wf_status launch_conv(const Schedule& S, const wf_conv_desc& d, const void* x, const void* packed,
                      const float* b_rep, void* y, wf_dtype out_dtype, uint32_t epilogue, cudaStream_t st,
                      int num_sms, std::string* err) {
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

  if (S.entries.size() > static_cast<size_t>(kMaxTable)) {
    *err = "schedule too long for the constant bank";
    return WF_UNSUPPORTED;
  }
  ConvArgs a;
  std::memset(&a, 0, sizeof(a));
  TmaMaps maps;
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
  a.box_bytes = Q * S.lbo_a;
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
    a.nt_col0[i] = t.col0;
    a.nt_cols[i] = t.cols;
    a.nt_bbytes[i] = static_cast<int>(t.b_bytes);
    a.nt_bsrc[i] = reinterpret_cast<long long>(packed_b + t.b_off);
    max_cols = std::max<uint32_t>(max_cols, static_cast<uint32_t>(t.cols));
  }
  const uint32_t fmt = (in_t == WF_BF16) ? 1u : (in_t == WF_F16 ? 0u : 2u);
  const uint32_t idesc_base = (1u << 4) | (fmt << 7) | (fmt << 10) | ((static_cast<uint32_t>(kTileM) >> 4) << 24);
  for (size_t i = 0; i < S.entries.size(); ++i) {
    const MmaEntry& e = S.entries[i];
    const uint32_t n8 = (e.meta >> 22) & 0x1FFu;  // N / 8 of this MMA
    const uint32_t lbo_b = n8 * 8u * 16u;         // B: [core col][N rows][16 B]
    a.table[i].x = (e.a_off >> 4) | ((static_cast<uint32_t>(S.lbo_a) >> 4) << 16);
    a.table[i].y = (e.b_off >> 4) | ((lbo_b >> 4) << 16);
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
  if (num_sms <= 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  a.ctas_per_ntile = std::max(1, std::min<int>(num_sms / a.n_tiles, a.num_mtiles));
  a.row_bytes = p.cout_f * oes;
  a.acc_stride = pow2ceil(max_cols);
  a.tmem_cols = 2 * a.acc_stride;
  a.epi_flags = static_cast<int>(epilogue);
  // shared-memory carve-up (offsets from the 1024-aligned base)
  a.off_a = 1024;
  a.off_b = a.off_a + a.stages * a.stage_bytes + kTileM * 16;
  a.off_b = (a.off_b + 127) / 128 * 128;
  a.off_bias = a.off_b + S.b_smem_bytes;
  const int smem = a.off_bias + kMaxAccCols * 4 + 1024;
  if (smem > kSmemLimit) {
    *err = "shared-memory budget exceeded";
    return WF_UNSUPPORTED;
  }

  // ---- input tensor maps (one 5-D view per H-stride residue) --------------------
  const int es = S.esize;
  const cuuint64_t rowpitch = static_cast<cuuint64_t>(d.w) * d.c * es;
  const cuuint64_t pix = static_cast<cuuint64_t>(p.f) * d.c * es;
  for (int b = 0; b < S.s; ++b) {
    if (!S.has_res[b]) continue;
    const cuuint64_t rows_b = static_cast<cuuint64_t>((d.h - b + S.s - 1) / S.s);
    cuuint64_t gdim[5] = {static_cast<cuuint64_t>(16 / es), static_cast<cuuint64_t>(p.wf), rows_b,
                          static_cast<cuuint64_t>(Q), static_cast<cuuint64_t>(d.n)};
    cuuint64_t gstr[4] = {pix, rowpitch * S.s, 16, rowpitch * d.h};
    cuuint32_t box[5] = {static_cast<cuuint32_t>(16 / es), static_cast<cuuint32_t>(p.wbox),
                         static_cast<cuuint32_t>(p.nrows), static_cast<cuuint32_t>(Q), 1};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    void* gaddr = const_cast<uint8_t*>(static_cast<const uint8_t*>(x) + b * rowpitch);
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
  cudaError_t e;
  const bool tf32 = (in_t == WF_TF32);
  if (tf32 && S.CH != 32) {
    *err = "tf32 plans use 32-column epilogue chunks";
    return WF_UNSUPPORTED;
  }
  if (out_dtype == WF_BF16)
    e = tf32 ? launch_typed<1, __nv_bfloat16, 32>(a, maps, grid, smem, st)
             : (S.CH == 64 ? launch_typed<0, __nv_bfloat16, 64>(a, maps, grid, smem, st)
                           : launch_typed<0, __nv_bfloat16, 32>(a, maps, grid, smem, st));
  else if (out_dtype == WF_F16)
    e = tf32 ? launch_typed<1, __half, 32>(a, maps, grid, smem, st)
             : (S.CH == 64 ? launch_typed<0, __half, 64>(a, maps, grid, smem, st)
                           : launch_typed<0, __half, 32>(a, maps, grid, smem, st));
  else
    e = tf32 ? launch_typed<1, float, 32>(a, maps, grid, smem, st)
             : (S.CH == 64 ? launch_typed<0, float, 64>(a, maps, grid, smem, st)
                           : launch_typed<0, float, 32>(a, maps, grid, smem, st));
  if (e != cudaSuccess) {
    *err = std::string("conv_fold_kernel launch failed: ") + cudaGetErrorString(e);
    return WF_CUDA_ERROR;
  }
  return WF_OK;
}

}  // namespace wfb
