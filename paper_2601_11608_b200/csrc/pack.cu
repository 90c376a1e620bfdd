// pack.cu -- K1: generalized block-diagonal filter expansion (SURVEY.md
// Appendix A), packed once into the tcgen05 B-operand layout, plus the dense
// expansion and bias replication.
//
// Reference: widthfold::expand_filter_general (src/fold.cpp:185-211) zero-fills
// a (KH,1,F*C,F*Cout) tensor and scatters w into the diagonal blocks; it throws
// for KW != 1 (src/fold.cpp:193-196). Here the expansion is generalized to
// KW > 1, stride and padding:
//   W'[kh, kw', fi*C + c, j*Cout + co] = w[kh, kw, c, co],
//   kw = (c0 + kw')*f + fi - j*s + pw   if 0 <= kw < KW, else exactly 0,
// and replicate_bias (src/fold.cpp:213-226) is b'[j*Cout + co] = b[co].
//
// Packed B layout, per schedule entry: a K-major, no-swizzle block
// [core col cc in {0,1}][n row (j,co) of the run][8 elems] (N*16 bytes per
// core column), i.e. exactly the smem descriptor layout the MMA reads
// (LBO = N*16, SBO = 128). Core column cc of the entry is the window-row core
// column c of filter row kh, nonzero for the accumulator slots in its mask
// (header words, plan.hpp Schedule::entry_cc0/1). Only the core columns a
// group's windows touch are stored.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "kernels.hpp"

namespace wfb {

struct PackArgs {
  int KH, KW, C, Cout, f, s, pw, c0, gs, Ng, E, esize, CH;
  int entries;
  int n_tiles;
  int nt_entry0[kMaxNTiles];
  int nt_g0[kMaxNTiles];
  long long nt_boff[kMaxNTiles];
  long long nt_bbytes[kMaxNTiles];
  int pair;  // 2: rows [0, N/2) of every block go to the first half of the N-tile's B, [N/2, N) to the second
  int n_groups;
  long long table_bytes;
  int round_tf32;
};

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <> __device__ __forceinline__ float to_f<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <> __device__ __forceinline__ float to_f<__half>(__half v) { return __half2float(v); }

// One CTA per schedule entry (run of accumulator slots, two core columns);
// threads walk its 2 core cols x N rows x (E/2) elements. Row nrow of the
// block is accumulator column slot0*Ng + nrow: group order[g0 + slot], output
// column chunk_perm(nrow % Ng) of that group.
template <typename T>
__global__ void pack_b_kernel(const T* __restrict__ w, uint8_t* __restrict__ packed, PackArgs a) {
  const int ei = blockIdx.x;
  const uint4 e = reinterpret_cast<const uint4*>(packed)[ei];
  const int* order = reinterpret_cast<const int*>(packed + 16LL * a.entries);
  const uint32_t* ccw = reinterpret_cast<const uint32_t*>(packed + 16LL * a.entries + 4LL * a.n_groups);
  const uint32_t cw[2] = {ccw[2 * ei], ccw[2 * ei + 1]};
  const int slot0 = (e.z >> 16) & 0x3f;
  const int N = static_cast<int>((e.z >> 22) & 0x1ffu) * 8;
  int nt = 0;
  while (nt + 1 < a.n_tiles && ei >= a.nt_entry0[nt + 1]) ++nt;
  const int half = a.E / 2;
  const int total = 2 * N * half;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int cc = idx / (N * half);
    int rem = idx - cc * N * half;
    const int nrow = rem / half;
    const int e8 = rem - nrow * half;
    const int kh = static_cast<int>(cw[cc] & 0xff);
    const int widx = static_cast<int>((cw[cc] >> 8) & 0xff) * half + e8;  // element of the KW'*f*C window row
    const int kp = widx / (a.f * a.C);
    const int r2 = widx - kp * a.f * a.C;
    const int fi = r2 / a.C;
    const int c = r2 - fi * a.C;
    const int g = order[a.nt_g0[nt] + slot0 + nrow / a.Ng];
    const int ncol = chunk_perm(nrow % a.Ng, a.CH);  // output column inside the group
    const int j = g * a.gs + ncol / a.Cout;
    const int co = ncol - (ncol / a.Cout) * a.Cout;
    const int kw = (a.c0 + kp) * a.f + fi - j * a.s + a.pw;
    const bool member = (cw[cc] >> (16 + nrow / a.Ng)) & 1u;  // this core column feeds the row's slot
    T val = T(0.0f);
    if (member && kw >= 0 && kw < a.KW) val = w[((static_cast<long long>(kh) * a.KW + kw) * a.C + c) * a.Cout + co];
    uint8_t* dst;
    if (a.pair == 2) {  // CTA r of the pair loads [nt_boff + r * b_bytes / 2, ...): its half of every block
      const int h = nrow / (N / 2), rr = nrow - h * (N / 2);
      dst = packed + a.table_bytes + a.nt_boff[nt] + h * (a.nt_bbytes[nt] / 2) + e.y / 2 + cc * (N / 2 * 16) +
            rr * 16 + e8 * a.esize;
    } else {
      dst = packed + a.table_bytes + a.nt_boff[nt] + e.y + cc * (N * 16) + nrow * 16 + e8 * a.esize;
    }
    if constexpr (sizeof(T) == 4) {
      float v = to_f(val);
      if (a.round_tf32) {
        uint32_t out;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(out) : "f"(v));
        v = __uint_as_float(out);
      }
      *reinterpret_cast<float*>(dst) = v;
    } else {
      *reinterpret_cast<T*>(dst) = val;
    }
  }
}

__global__ void replicate_bias_kernel(const float* __restrict__ b, float* __restrict__ out, int Cout, int r) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < Cout * r) out[i] = b[i % Cout];
}

// Dense W'(KH, KW', f*C, r*Cout): one thread per output element, fp32 bits moved exactly.
__global__ void expand_dense_kernel(const float* __restrict__ w, float* __restrict__ out, int KH, int KW, int C,
                                    int Cout, int f, int s, int pw, int c0, int kwf, int r) {
  const long long Cif = (long long)f * C, Cof = (long long)r * Cout;
  const long long total = (long long)KH * kwf * Cif * Cof;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    long long t = idx;
    const int n = static_cast<int>(t % Cof); t /= Cof;
    const int k = static_cast<int>(t % Cif); t /= Cif;
    const int kp = static_cast<int>(t % kwf); t /= kwf;
    const int kh = static_cast<int>(t);
    const int fi = k / C, c = k % C, j = n / Cout, co = n % Cout;
    const int kw = (c0 + kp) * f + fi - j * s + pw;
    out[idx] = (kw >= 0 && kw < KW) ? w[((static_cast<long long>(kh) * KW + kw) * C + c) * Cout + co] : 0.0f;
  }
}

wf_status launch_pack(const Schedule& S, const wf_conv_desc& d, const void* w, const float* b, void* packed,
                      float* b_rep, cudaStream_t st, std::string* err) {
  note_operand_write();  // the next conv launch must not overlap this write (programmatic dependent launch)
  const wf_fold_plan& p = S.plan;
  // schedule table first: the pack kernel and the conv kernel both read it.
  // header = schedule table + slot order. A pageable-source cudaMemcpyAsync
  // returns once the bytes are staged, so the temporary may go out of scope.
  std::vector<uint8_t> header(static_cast<size_t>(p.table_bytes), 0);
  std::memcpy(header.data(), S.entries.data(), S.entries.size() * sizeof(MmaEntry));
  std::memcpy(header.data() + S.entries.size() * sizeof(MmaEntry), S.order.data(), S.order.size() * sizeof(int));
  if (S.entry_cc0.size() != S.entries.size() || S.entry_cc1.size() != S.entries.size()) {
    *err = "pack: schedule has no core-column words";
    return WF_INVALID_ARGUMENT;
  }
  {
    uint32_t* ccw = reinterpret_cast<uint32_t*>(header.data() + S.entries.size() * sizeof(MmaEntry) +
                                                S.order.size() * sizeof(int));
    for (size_t i = 0; i < S.entries.size(); ++i) {
      ccw[2 * i] = S.entry_cc0[i];
      ccw[2 * i + 1] = S.entry_cc1[i];
    }
  }
  cudaError_t e = cudaMemsetAsync(packed, 0, static_cast<size_t>(p.packed_bytes), st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(packed, header.data(), header.size(), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) {
    *err = std::string("pack: table upload failed: ") + cudaGetErrorString(e);
    return WF_CUDA_ERROR;
  }
  PackArgs a{};
  a.KH = static_cast<int>(d.kh);
  a.KW = static_cast<int>(d.kw);
  a.C = static_cast<int>(d.c);
  a.Cout = static_cast<int>(d.cout);
  a.f = static_cast<int>(p.f);
  a.s = static_cast<int>(d.stride_w);
  a.pw = static_cast<int>(d.pad_w);
  a.c0 = static_cast<int>(p.c0);
  a.gs = static_cast<int>(p.group_size);
  a.Ng = S.Ng;
  a.E = S.E;
  a.esize = S.esize;
  a.CH = S.CH;
  a.pair = S.pair;
  a.n_groups = static_cast<int>(S.order.size());
  a.entries = static_cast<int>(S.entries.size());
  a.n_tiles = static_cast<int>(S.ntiles.size());
  for (int i = 0; i < a.n_tiles; ++i) {
    a.nt_entry0[i] = S.ntiles[i].entry0;
    a.nt_g0[i] = S.ntiles[i].g0;
    a.nt_boff[i] = S.ntiles[i].b_off;
    a.nt_bbytes[i] = S.ntiles[i].b_bytes;
  }
  a.table_bytes = p.table_bytes;
  a.round_tf32 = 1;
  const int blocks = a.entries;
  const int threads = 256;
  const wf_dtype t = static_cast<wf_dtype>(p.in_dtype);
  if (t == WF_BF16)
    pack_b_kernel<__nv_bfloat16><<<blocks, threads, 0, st>>>(static_cast<const __nv_bfloat16*>(w),
                                                             static_cast<uint8_t*>(packed), a);
  else if (t == WF_F16)
    pack_b_kernel<__half><<<blocks, threads, 0, st>>>(static_cast<const __half*>(w), static_cast<uint8_t*>(packed), a);
  else
    pack_b_kernel<float><<<blocks, threads, 0, st>>>(static_cast<const float*>(w), static_cast<uint8_t*>(packed), a);
  e = cudaGetLastError();
  if (e == cudaSuccess && b_rep != nullptr) {
    const int n = static_cast<int>(p.cout_f);
    if (b != nullptr)
      replicate_bias_kernel<<<(n + 255) / 256, 256, 0, st>>>(b, b_rep, static_cast<int>(d.cout), static_cast<int>(p.r));
    else
      e = cudaMemsetAsync(b_rep, 0, n * sizeof(float), st);
    if (e == cudaSuccess) e = cudaGetLastError();
  }
  if (e != cudaSuccess) {
    *err = std::string("pack kernel failed: ") + cudaGetErrorString(e);
    return WF_CUDA_ERROR;
  }
  return WF_OK;
}

wf_status launch_replicate_bias(const float* b, int cout, int r, float* out, cudaStream_t st, std::string* err) {
  note_operand_write();
  replicate_bias_kernel<<<(cout * r + 255) / 256, 256, 0, st>>>(b, out, cout, r);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("replicate_bias_kernel: ") + cudaGetErrorString(e);
    return WF_CUDA_ERROR;
  }
  return WF_OK;
}

wf_status launch_expand_dense(const wf_conv_desc& d, int64_t f, const float* w, float* out, cudaStream_t st,
                              std::string* err) {
  const int64_t s = d.stride_w;
  const int64_t r = f / s;
  const int64_t c0 = -((d.pad_w + f - 1) / f);
  int64_t num = f - s - d.pad_w + d.kw - 1;
  int64_t fl = num / f;
  if ((num % f != 0) && (num < 0)) --fl;
  const int64_t kwf = fl - c0 + 1;
  const long long total = (long long)d.kh * kwf * f * d.c * r * d.cout;
  const int threads = 256;
  const int blocks = static_cast<int>(std::min<long long>((total + threads - 1) / threads, 8192));
  expand_dense_kernel<<<blocks, threads, 0, st>>>(w, out, (int)d.kh, (int)d.kw, (int)d.c, (int)d.cout, (int)f, (int)s,
                                                  (int)d.pad_w, (int)c0, (int)kwf, (int)r);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("expand kernel failed: ") + cudaGetErrorString(e);
    return WF_CUDA_ERROR;
  }
  return WF_OK;
}

}  // namespace wfb
