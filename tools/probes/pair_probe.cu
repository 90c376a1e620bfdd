// Probe: tcgen05.mma issue cost, cta_group::1 (M=128) vs cta_group::2
// (M=256 over a CTA pair), SS operands, no swizzle, for N = 64/128/256.
// Prints cycles per MMA measured by the issuing thread (commit + wait).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2601_11608_b200/csrc/ptx.cuh"
using namespace wfb::ptx;

template <int kPair>
__global__ void __cluster_dims__(kPair, 1, 1) __launch_bounds__(128, 1)
    probe(int N, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = (kPair == 2) ? cluster_ctarank() : 0;
  const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_barrier_init(); }
  if (warp == 0) {
    if (kPair == 2) tmem_alloc_pair(smem_u32(&tslot), 512);
    else tmem_alloc(smem_u32(&tslot), 512);
  }
  asm volatile("fence.proxy.async.shared::cta;");
  tc_fence_before();
  if (kPair == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u * kPair >> 4) << 24);
  const uint64_t ad = smem_desc(base, 128 * 16, 128);
  const uint64_t bd = smem_desc(base + 64 * 1024, (N / kPair) * 16, 128);
  if (warp == 1 && rank == 0) {
    const bool leader = elect_one();
    __syncwarp();
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (leader) {
        if (kPair == 2) mma_pair(tmem + (i & 1) * 256, ad + 2 * (i & 7), bd + 2 * (i & 7), idesc, 1);
        else mma<0>(tmem + (i & 1) * 256, ad + 2 * (i & 7), bd + 2 * (i & 7), idesc, 1);
      }
    }
    if (leader) {
      if (kPair == 2) mma_commit_pair(smem_u32(&bar), 0x1);
      else mma_commit(smem_u32(&bar));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  if (kPair == 2) cluster_sync(); else __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    if (kPair == 2) tmem_dealloc_pair(tmem, 512); else tmem_dealloc(tmem, 512);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 148);
  cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 4096;
  printf("pair  N  cycles/MMA (per pair in pair mode; 1-CTA M=128 ideal N/2, pair M=256 ideal N/2 per SM)\n");
  for (int pair : {1, 2})
    for (int N : {32, 64, 128, 256}) {
      if (pair == 2 && N < 64) continue;
      if (pair == 1) probe<1><<<148, 128, 100 * 1024>>>(N, iters, d);
      else probe<2><<<148, 128, 100 * 1024>>>(N, iters, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      unsigned long long h;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("%4d %3d  %8.1f\n", pair, N, (double)h / iters);
    }
  return 0;
}
