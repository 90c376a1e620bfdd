// aux_kernels.cu -- the non-hot-path device operations behind the reference API.
//
//   conv_direct_kernel   widthfold::conv2d (src/refconv.cpp:34-80) bit-for-bit:
//                        fp32, per output element kh -> kw -> ci, separately
//                        rounded multiply and add (no FMA), accumulator +0.0f,
//                        plus explicit zero padding. Used for the reference's
//                        exact-fp32 semantics (precision="exact") and for
//                        grouped_conv (src/blockdiag.cpp:138-187), which the
//                        reference guarantees bitwise equal to the dense conv.
//   bias_add_kernel      widthfold::bias_add (src/refconv.cpp:82-95) (+ReLU).
//   repitch_kernel       the device fold for rows whose pitch is not a 16-byte
//                        multiple or whose width is not a multiple of f
//                        (AlexNet: W=227, 1362-byte rows): copies x into a
//                        workspace of pitch Wp*C (zero tail) so the folded view
//                        is again a TMA-addressable reshape.
//   blockdiag_check      BlockDiagFilter::from_expanded's strict-zero check
//                        (src/blockdiag.cpp:24-84): any off-diagonal entry that
//                        is not +-0.0f is an error.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <type_traits>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <string>

#include "kernels.hpp"

namespace wfb {

// One warp per row (grid-stride over rows). Lane L of a round owns output
// chunk k = base + L = input-row bytes [16k, 16k+16): it loads the aligned
// 16-byte chunk k of the row's aligned superset once (coalesced, 512 B per
// warp-round), takes chunk k+1 from lane L+1 by shuffle (lane 31 from lane 0
// of the next round),
// and funnel-shifts the pair by the row's misalignment -- every input byte is
// read once and every output byte written once. Bytes past rb_in are zero.
// Bytes [4*Q4 + bs/8, +16) of the 32-byte pair (a, b): the row's word offset
// Q4 is a template parameter (uniform per row), so no indexed selects.
template <int Q4>
__device__ __forceinline__ void shift_out(const uint4& a, const uint4& b, uint32_t bs, uint32_t (&w)[4]) {
  const uint32_t q[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
  for (int t = 0; t < 4; ++t) w[t] = __funnelshift_r(q[t + Q4], q[t + Q4 + 1], bs);  // bs = 0: q[t + Q4]
}

// One row's chunks, loaded (kRounds rounds of 32 + the chunk after them for
// lane 0, all in flight at once) and then shifted and stored: lane 31's right
// neighbour comes from lane 0 of the next round by shuffle, so no load waits
// on another. Rows shorter than 32 * kRounds chunks take one round trip.
constexpr int kRepitchRounds = 3;
struct RowChunks {
  uint4 c[kRepitchRounds + 1];
};

__device__ __forceinline__ void repitch_load(const uint4* a0, int s0, int nin, int lane, bool valid, RowChunks& rc) {
  const uint4 z = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
  for (int j = 0; j <= kRepitchRounds; ++j) {
    const int k = s0 + 32 * j + lane;
    rc.c[j] = (valid && k < nin && (j < kRepitchRounds || lane == 0)) ? __ldg(a0 + k) : z;
  }
}

// Output chunk k of a row goes to byte 16k (row layout) or, with Q core-column
// planes (plane layout), to plane k % Q at column k / Q: [q][folded col][16 B],
// each plane plane_bytes long, so the TMA boxes of the conv read whole
// folded-column runs of one core column (up to 512-byte pieces) instead of
// 16-byte ones.
__device__ __forceinline__ int chunk_dst(int k, int Q, int plane_bytes) {
  return Q > 0 ? (k % Q) * plane_bytes + (k / Q) * 16 : 16 * k;
}

template <int Q4>
__device__ __forceinline__ void repitch_store(const RowChunks& rc, uint8_t* dst, int s0, int cpr, int rb_in,
                                              uint32_t bs, int lane, int Q, int plane_bytes) {
#pragma unroll
  for (int j = 0; j < kRepitchRounds; ++j) {
    const int k = s0 + 32 * j + lane;
    const int src = (lane + 1) & 31;
    uint4 n;
    n.x = __shfl_sync(0xffffffffu, (lane == 0) ? rc.c[j + 1].x : rc.c[j].x, src);
    n.y = __shfl_sync(0xffffffffu, (lane == 0) ? rc.c[j + 1].y : rc.c[j].y, src);
    n.z = __shfl_sync(0xffffffffu, (lane == 0) ? rc.c[j + 1].z : rc.c[j].z, src);
    n.w = __shfl_sync(0xffffffffu, (lane == 0) ? rc.c[j + 1].w : rc.c[j].w, src);
    if (k >= cpr) continue;
    uint32_t w[4];
    shift_out<Q4>(rc.c[j], n, bs, w);
    const int o = 16 * k;
    if (o + 16 > rb_in) {  // zero the bytes past the input row
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        uint32_t m = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (o + 4 * t + b < rb_in) m |= 0xFFu << (8 * b);
        w[t] &= m;
      }
    }
    *reinterpret_cast<uint4*>(dst + chunk_dst(k, Q, plane_bytes)) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

__device__ __forceinline__ void repitch_store_any(const RowChunks& rc, uint8_t* dst, int s0, int cpr, int rb_in,
                                                  int sh, int lane, int Q, int plane_bytes) {
  const uint32_t bs = static_cast<uint32_t>(sh & 3) * 8;
  switch (sh >> 2) {  // warp-uniform
    case 0: repitch_store<0>(rc, dst, s0, cpr, rb_in, bs, lane, Q, plane_bytes); break;
    case 1: repitch_store<1>(rc, dst, s0, cpr, rb_in, bs, lane, Q, plane_bytes); break;
    case 2: repitch_store<2>(rc, dst, s0, cpr, rb_in, bs, lane, Q, plane_bytes); break;
    default: repitch_store<3>(rc, dst, s0, cpr, rb_in, bs, lane, Q, plane_bytes); break;
  }
}

// Two rows per warp in flight (grid-stride pairs of rows). (Assembling the plane
// layout's rows in shared memory to store them contiguously measured slower
// than these scattered 16-byte stores: AlexNet b512 73 vs 61 us.)
__global__ void __launch_bounds__(256) repitch_kernel(const uint8_t* __restrict__ x, uint8_t* __restrict__ y,
                                                      long long rows, int rb_in, int rb_out, int Q, int plane_bytes,
                                                      int rev) {
  const int lane = threadIdx.x & 31;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  const int cpr = rb_out >> 4;
  for (long long r = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < rows;
       r += 2 * nwarps) {
    const bool has2 = r + nwarps < rows;
    // rev: rows in descending order, so the rows written last (still in L2) are the first the conv reads
    const long long ra = rev ? rows - 1 - r : r;
    const long long r2 = has2 ? (rev ? rows - 1 - (r + nwarps) : r + nwarps) : ra;
    const uintptr_t src = reinterpret_cast<uintptr_t>(x) + ra * rb_in;
    const uintptr_t src2 = reinterpret_cast<uintptr_t>(x) + r2 * rb_in;
    const uint4* a0 = reinterpret_cast<const uint4*>(src & ~static_cast<uintptr_t>(15));
    const uint4* a2 = reinterpret_cast<const uint4*>(src2 & ~static_cast<uintptr_t>(15));
    const int sh = static_cast<int>(src & 15u), sh2 = static_cast<int>(src2 & 15u);
    const int nin = (sh + rb_in + 15) >> 4, nin2 = (sh2 + rb_in + 15) >> 4;  // aligned chunks holding the row
    uint8_t* const d1 = y + ra * rb_out;
    uint8_t* const d2 = y + r2 * rb_out;
    for (int s0 = 0; s0 < cpr; s0 += 32 * kRepitchRounds) {
      RowChunks c1, c2;
      repitch_load(a0, s0, nin, lane, true, c1);
      repitch_load(a2, s0, nin2, lane, has2, c2);
      repitch_store_any(c1, d1, s0, cpr, rb_in, sh, lane, Q, plane_bytes);
      if (has2) repitch_store_any(c2, d2, s0, cpr, rb_in, sh2, lane, Q, plane_bytes);
    }
  }
}

static int repitch_reverse() {
  static const int rev = [] {
    const char* e = std::getenv("WF_REPITCH_REV");
    return (e && e[0] == '1') ? 1 : 0;
  }();
  return rev;
}

wf_status launch_repitch(const void* x, void* ws, long long rows, int rb_in, int rb_out, int planes,
                         cudaStream_t st, std::string* err) {
  const int threads = 256;  // 8 warps, one row each at a time
  const int blocks = static_cast<int>(std::min<long long>((rows + 7) / 8, 148LL * 8));
  repitch_kernel<<<blocks, threads, 0, st>>>(static_cast<const uint8_t*>(x), static_cast<uint8_t*>(ws), rows, rb_in,
                                             rb_out, planes, planes > 0 ? rb_out / planes : 0, repitch_reverse());
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("repitch_kernel: ") + cudaGetErrorString(e);
    return WF_CUDA_ERROR;
  }
  return WF_OK;
}

__global__ void conv_direct_kernel(const float* __restrict__ x, const float* __restrict__ w, float* __restrict__ y,
                                   int B, int H, int W, int C, int KH, int KW, int Co, int sh, int sw, int ph,
                                   int pw, int OH, int OW, int groups) {
  // groups > 1: the grouped conv of a block-diagonal dense filter -- output
  // channel oc reads only the input channels of its own block, in the same
  // kh -> kw -> ci order (src/blockdiag.cpp:138-187), so skipped terms are
  // never formed (no 0 * NaN) and the surviving sum is the dense one's.
  const int Cib = C / groups, Cob = Co / groups;
  const long long total = (long long)B * OH * OW * Co;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    long long t = idx;
    const int oc = static_cast<int>(t % Co); t /= Co;
    const int ow = static_cast<int>(t % OW); t /= OW;
    const int oh = static_cast<int>(t % OH); t /= OH;
    const int b = static_cast<int>(t);
    float acc = 0.0f;
    for (int kh = 0; kh < KH; ++kh) {
      const int ih = oh * sh - ph + kh;
      for (int kw = 0; kw < KW; ++kw) {
        const int iw = ow * sw - pw + kw;
        const bool in = (ih >= 0 && ih < H && iw >= 0 && iw < W);
        const float* xr = x + (((long long)b * H + (in ? ih : 0)) * W + (in ? iw : 0)) * C;
        const float* wr = w + ((long long)(kh * KW + kw) * C) * Co + oc;
        const int c_lo = (oc / Cob) * Cib;
        for (int ci = c_lo; ci < c_lo + Cib; ++ci) {
          const float xv = in ? xr[ci] : 0.0f;
          acc = __fadd_rn(acc, __fmul_rn(xv, wr[(long long)ci * Co]));
        }
      }
    }
    y[idx] = acc;
  }
}

__global__ void bias_add_kernel(const float* __restrict__ y, const float* __restrict__ b, float* __restrict__ out,
                                long long n, int C, int relu) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float v = __fadd_rn(y[i], b[i % C]);
    if (relu && v < 0.0f) v = 0.0f;
    out[i] = v;
  }
}

__global__ void blockdiag_check_kernel(const float* __restrict__ wd, int KH, int KW, int Cif, int Cof, int groups,
                                       unsigned long long* __restrict__ first_bad) {
  const long long total = (long long)KH * KW * Cif * Cof;
  const int Cib = Cif / groups, Cob = Cof / groups;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int co = static_cast<int>(i % Cof);
    const int ci = static_cast<int>((i / Cof) % Cif);
    if (co / Cob != ci / Cib && wd[i] != 0.0f) atomicMin(first_bad, static_cast<unsigned long long>(i));
  }
}

static int grid_for(long long total) {
  const long long g = (total + 255) / 256;
  return static_cast<int>(g < 1 ? 1 : (g > 65535 ? 65535 : g));
}

wf_status launch_conv_direct(const wf_conv_desc& d, const float* x, const float* w, float* y, int groups,
                             cudaStream_t st, std::string* err) {
  const int64_t OH = (d.h + 2 * d.pad_h - d.kh) / d.stride_h + 1;
  const int64_t OW = (d.w + 2 * d.pad_w - d.kw) / d.stride_w + 1;
  const long long total = (long long)d.n * OH * OW * d.cout;
  conv_direct_kernel<<<grid_for(total), 256, 0, st>>>(x, w, y, (int)d.n, (int)d.h, (int)d.w, (int)d.c, (int)d.kh,
                                                      (int)d.kw, (int)d.cout, (int)d.stride_h, (int)d.stride_w,
                                                      (int)d.pad_h, (int)d.pad_w, (int)OH, (int)OW, groups);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("conv_direct_kernel: ") + cudaGetErrorString(e);
    return WF_CUDA_ERROR;
  }
  return WF_OK;
}

wf_status launch_bias_add(const float* y, const float* b, float* out, long long n, int C, int relu, cudaStream_t st,
                          std::string* err) {
  bias_add_kernel<<<grid_for(n), 256, 0, st>>>(y, b, out, n, C, relu);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("bias_add_kernel: ") + cudaGetErrorString(e);
    return WF_CUDA_ERROR;
  }
  return WF_OK;
}

// fp32 -> bf16 / fp16, round to nearest even (the device dtypes of a folded graph node)
template <typename T>
__global__ void cast_f32_kernel(const float* __restrict__ x, T* __restrict__ y, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    if constexpr (sizeof(T) == 2 && std::is_same<T, __nv_bfloat16>::value) y[i] = __float2bfloat16_rn(x[i]);
    else y[i] = __float2half_rn(x[i]);
  }
}

wf_status launch_cast_f32(const float* x, void* y, long long n, wf_dtype to, cudaStream_t st, std::string* err) {
  if (to == WF_BF16)
    cast_f32_kernel<__nv_bfloat16><<<grid_for(n), 256, 0, st>>>(x, static_cast<__nv_bfloat16*>(y), n);
  else if (to == WF_F16)
    cast_f32_kernel<__half><<<grid_for(n), 256, 0, st>>>(x, static_cast<__half*>(y), n);
  else {
    *err = "cast: target dtype must be bf16 or f16";
    return WF_INVALID_ARGUMENT;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("cast_f32_kernel: ") + cudaGetErrorString(e);
    return WF_CUDA_ERROR;
  }
  return WF_OK;
}

wf_status launch_blockdiag_check(const float* wd, int KH, int KW, int Cif, int Cof, int groups,
                                 unsigned long long* scratch, long long* first_bad, cudaStream_t st, std::string* err) {
  const unsigned long long init = ~0ull;
  cudaError_t e = cudaMemcpyAsync(scratch, &init, sizeof(init), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) {
    const long long total = (long long)KH * KW * Cif * Cof;
    blockdiag_check_kernel<<<grid_for(total), 256, 0, st>>>(wd, KH, KW, Cif, Cof, groups, scratch);
    e = cudaGetLastError();
  }
  unsigned long long h = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, scratch, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    *err = std::string("blockdiag check: ") + cudaGetErrorString(e);
    return WF_CUDA_ERROR;
  }
  *first_bad = (h == ~0ull) ? -1 : static_cast<long long>(h);
  return WF_OK;
}

}  // namespace wfb
