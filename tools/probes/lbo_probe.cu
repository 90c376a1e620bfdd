// Probe: does a "negative" leading-byte-offset (core column 1 stored BELOW
// core column 0, LBO encoded modulo 2^14 x 16 B) work in a tcgen05 smem
// descriptor? D(128x64) = A(128x16) * B(16x64), B = [I16; 0], so D[:, :16]
// must equal A. Prints the number of mismatches for LBO > 0 and LBO < 0.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2601_11608_b200/csrc/ptx.cuh"
using namespace wfb::ptx;

__global__ void probe(int neg, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
  uint8_t* g = smem + (base - smem_u32(smem));
  // A core columns: kc=0 at offA0, kc=1 at offA1
  const uint32_t offA0 = neg ? 4096 : 0, offA1 = neg ? 0 : 4096, offB = 8192;
  for (int m = threadIdx.x; m < 128; m += blockDim.x)
    for (int k = 0; k < 16; ++k) {
      const uint32_t off = (k < 8 ? offA0 : offA1) + (m / 8) * 128 + (m % 8) * 16 + (k % 8) * 2;
      *reinterpret_cast<__nv_bfloat16*>(g + off) = __float2bfloat16(static_cast<float>((m * 3 + k) % 61));
    }
  for (int n = threadIdx.x; n < 64; n += blockDim.x)
    for (int k = 0; k < 16; ++k) {
      const uint32_t off = offB + (k / 8) * 1024 + (n / 8) * 128 + (n % 8) * 16 + (k % 8) * 2;
      *reinterpret_cast<__nv_bfloat16*>(g + off) = __float2bfloat16(n == k ? 1.0f : 0.0f);
    }
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(smem_u32(&tslot), 64);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 1) {
    const int32_t lbo = static_cast<int32_t>(offA1) - static_cast<int32_t>(offA0);
    const uint32_t lbo_field = static_cast<uint32_t>(lbo >> 4) & 0x3FFFu;  // modulo 2^14 units
    const uint64_t ad = static_cast<uint64_t>(((base + offA0) >> 4) & 0x3FFFu) | (static_cast<uint64_t>(lbo_field) << 16) |
                        (static_cast<uint64_t>(128 >> 4) << 32) | (1ull << 46);
    const uint64_t bd = smem_desc(base + offB, 1024, 128);
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
    if (elect_one()) {
      mma<0>(tmem, ad, bd, idesc, 0);
      mma_commit(smem_u32(&bar));
    }
    __syncwarp();
  }
  mbar_wait(smem_u32(&bar), 0);
  tc_fence_after();
  uint32_t r[16];
  tmem_ld16(tmem + ((32u * warp) << 16), r);
  tmem_ld_wait();
  for (int c = 0; c < 16; ++c) out[(32 * warp + lane) * 16 + c] = __uint_as_float(r[c]);
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 64); }
}

int main() {
  float* d; cudaMalloc(&d, 128 * 16 * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 1024);
  for (int neg = 0; neg < 2; ++neg) {
    cudaMemset(d, 0, 128 * 16 * 4);
    probe<<<1, 128, 16384 + 1024>>>(neg, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("neg=%d err %s\n", neg, cudaGetErrorString(e)); return 1; }
    float h[128 * 16];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < 128; ++m)
      for (int k = 0; k < 16; ++k) bad += h[m * 16 + k] != static_cast<float>((m * 3 + k) % 61);
    printf("LBO %s: %d mismatches of 2048 (D[5][9] = %g, want %d)\n", neg ? "negative (mod 2^14)" : "positive", bad,
           h[5 * 16 + 9], (5 * 3 + 9) % 61);
  }
  return 0;
}
