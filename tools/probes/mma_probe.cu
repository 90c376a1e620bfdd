// Microbenchmark: tcgen05.mma (kind::f16, M=128, K=16, SS) issue throughput on
// one SM vs N, smem layout (no swizzle / 128B swizzle), A start alignment, and
// accumulator dependency. Prints cycles per MMA.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2601_11608_b200/csrc/ptx.cuh"
using namespace wfb::ptx;

__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}

template <int reuse>
__global__ void __launch_bounds__(128, 1) probe(int N, int layout, int a_shift, int nacc, int iters,
                                               unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(smem_u32(&tslot), 512);
  asm volatile("fence.proxy.async.shared::cta;");
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
  unsigned long long t0 = 0, t1 = 0;
  const int wu = __shfl_sync(0xffffffff, warp, 0);
  if (wu == 1) {
    const uint32_t a0 = base + a_shift;          // A: 128 rows
    const uint32_t b0 = base + 64 * 1024;        // B: N rows
    uint64_t ad, bd;
    if (layout == 0) {  // no swizzle, K-major: core 8x16B, SBO=128, LBO = rows*16
      ad = desc(a0, 128 * 16, 128, 0);
      bd = desc(b0, N * 16, 128, 0);
    } else {            // 128B swizzle K-major: rows of 128B (64 bf16), SBO = 1024
      ad = desc(a0, 16, 1024, 2);
      bd = desc(b0, 16, 1024, 2);
    }
    const uint32_t accstride = (uint32_t)N;
    const bool leader = elect_one();
    __syncwarp();
    t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t d = tmem + (uint32_t)((j % nacc) * accstride);
        if constexpr (reuse) {
          if (leader) {
            if ((j % 4) == 0) mma_coll<0>(d, ad, bd + 2 * j, idesc, j != 0, 1);
            else if ((j % 4) == 3) mma_coll<0>(d, ad, bd + 2 * j, idesc, j != 0, 3);
            else mma_coll<0>(d, ad, bd + 2 * j, idesc, j != 0, 2);
          }
        } else {
          if (leader) mma<0>(d, ad + 2 * (j & 1), bd + 2 * j, idesc, j != 0);
        }
      }
    }
    if (leader) mma_commit(smem_u32(&bar));
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
    t1 = clock64();
    if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 8 * 148);
  cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 170 * 1024);
  cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 170 * 1024);
  const int iters = 4096;
  printf("grid  N  layout reuseA nacc  cyc/mma   (ideal M128 = N/2)\n");
  for (int grid : {148})
  for (int layout : {0, 2})
  for (int N : {32, 64, 128, 256})
  for (int reuse : {0, 1})
  for (int nacc : {1}) {
    const int a_shift = 0;
    if (reuse) probe<1><<<grid, 128, 170 * 1024>>>(N, layout, a_shift, nacc, iters, d);
    else probe<0><<<grid, 128, 170 * 1024>>>(N, layout, a_shift, nacc, iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%4d %3d %6d %6d %4d  %8.1f\n", grid, N, layout, reuse, nacc, (double)h / iters);
  }
  return 0;
}
