// Probe: a K-major SWIZZLE_32B A operand (rows of 32 bytes = one K=16 step,
// 16-byte halves XOR-swizzled by address bit 7) read through descriptors whose
// start address is shifted by s rows (the im2col row-shift trick). Which
// base_offset encoding (if any) makes every shift correct?
// D(128x64) = A(128x16) * B, B = [I16; 0]  =>  D[:, :16] must equal A.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2601_11608_b200/csrc/ptx.cuh"
using namespace wfb::ptx;

__global__ void probe(int s, int mode, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
  uint8_t* g = smem + (base - smem_u32(smem));
  const uint32_t offB = 16384;
  // A rows R = 0..143, logical address 32R + 2k, physical: bit4 ^= bit7
  for (int R = threadIdx.x; R < 144; R += blockDim.x)
    for (int k = 0; k < 16; ++k) {
      uint32_t L = 32 * R + 2 * k;
      uint32_t P = L ^ (((L >> 7) & 1u) << 4);
      *reinterpret_cast<__nv_bfloat16*>(g + P) = __float2bfloat16(static_cast<float>((R * 3 + k) % 61));
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
    const uint32_t start = base + 32 * s;
    uint64_t bo = 0;
    if (mode == 1) bo = (start >> 7) & 7;
    if (mode == 2) bo = (start >> 8) & 7;
    if (mode == 3) bo = (start >> 5) & 7;
    const uint64_t ad = static_cast<uint64_t>((start >> 4) & 0x3FFFu) | (1ull << 16) |
                        (static_cast<uint64_t>(256 >> 4) << 32) | (1ull << 46) | (bo << 49) | (6ull << 61);
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
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 24 * 1024);
  printf("shift  mode0(bo=0)  mode1(bo=addr>>7&7)  mode2(addr>>8&7)  mode3(addr>>5&7)   [mismatches of 2048]\n");
  for (int s : {0, 1, 2, 3, 4, 5, 7, 8, 9, 12}) {
    printf("%5d", s);
    for (int mode = 0; mode < 4; ++mode) {
      cudaMemset(d, 0, 128 * 16 * 4);
      probe<<<1, 128, 24 * 1024>>>(s, mode, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("  err %s\n", cudaGetErrorString(e)); return 1; }
      float h[128 * 16];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int m = 0; m < 128; ++m)
        for (int k = 0; k < 16; ++k) bad += h[m * 16 + k] != static_cast<float>(((m + s) * 3 + k) % 61);
      printf("  %12d", bad);
    }
    printf("\n");
  }
  return 0;
}
