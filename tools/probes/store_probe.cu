// store_probe.cu -- energy of the output-write paths the conv epilogue could use.
//
// Each variant writes `bytes` of a device buffer (13.15 GB = R50 conv1 b8192's
// bf16 output) from data already on chip:
//   0  st.global.v8   (32 B per thread per store, the epilogue's instruction)
//   1  st.global.v4   (16 B)
//   2  cp.async.bulk.global.shared::cta (TMA bulk store) of 16 KB chunks from a
//      shared-memory buffer filled once, 4 chunks in flight per CTA
//   3  st.global.v8 with L1::no_allocate + L2::evict_first
// Persistent grids (148 x k CTAs). tools/store_probe.py times each in a loop
// and samples board power: mJ per GB under the 1000 W cap decides whether a
// TMA-store epilogue would buy energy back.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
//        -o tools/probes/libstore_probe.so tools/probes/store_probe.cu
#include <cuda_runtime.h>

#include <cstdint>

namespace {

__global__ void __launch_bounds__(256) st_v8(uint8_t* __restrict__ y, long long bytes, uint32_t seed) {
  const long long n32 = bytes >> 5;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  uint32_t v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = seed * (threadIdx.x + 1) + k;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n32; i += stride)
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(y + 32 * i), "r"(v[0]), "r"(v[1]),
                 "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

__global__ void __launch_bounds__(256) st_v8_stream(uint8_t* __restrict__ y, long long bytes, uint32_t seed) {
  const long long n32 = bytes >> 5;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  uint32_t v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = seed * (threadIdx.x + 1) + k;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n32; i += stride)
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(
                     y + 32 * i),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

__global__ void __launch_bounds__(256) st_v4(uint8_t* __restrict__ y, long long bytes, uint32_t seed) {
  const long long n16 = bytes >> 4;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  const uint4 v = make_uint4(seed * threadIdx.x, seed + 1, seed + 2, seed + 3);
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += stride)
    asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(y + 16 * i), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}

constexpr int kChunk = 16384;
constexpr int kInFlight = 4;

__global__ void __launch_bounds__(128) bulk_store(uint8_t* __restrict__ y, long long bytes, uint32_t seed) {
  extern __shared__ __align__(128) uint8_t sbuf[];
  for (int i = threadIdx.x; i < kChunk * kInFlight / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sbuf)[i] = seed * (i + 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  const long long nchunks = bytes / kChunk;
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(sbuf));
  int k = 0;
  for (long long c = blockIdx.x; c < nchunks; c += gridDim.x, ++k) {
    if (k >= kInFlight) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kInFlight - 1) : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(y + c * kChunk),
                 "r"(s + (k % kInFlight) * kChunk), "r"(kChunk)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

}  // namespace

extern "C" int store_probe(int variant, void* y, long long bytes, int sms, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  static uint32_t seed = 1;
  ++seed;
  switch (variant) {
    case 0: st_v8<<<sms * 8, 256, 0, st>>>(static_cast<uint8_t*>(y), bytes, seed); break;
    case 1: st_v4<<<sms * 8, 256, 0, st>>>(static_cast<uint8_t*>(y), bytes, seed); break;
    case 2: {
      const int smem = kChunk * kInFlight;
      cudaFuncSetAttribute(bulk_store, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      bulk_store<<<sms * 3, 128, smem, st>>>(static_cast<uint8_t*>(y), bytes, seed);
      break;
    }
    case 3: st_v8_stream<<<sms * 8, 256, 0, st>>>(static_cast<uint8_t*>(y), bytes, seed); break;
    default: return -1;
  }
  return static_cast<int>(cudaGetLastError());
}
