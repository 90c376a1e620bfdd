// Probe: thread <-> (TMEM lane, column) mapping of tcgen05.ld.16x256b.
// Writes lane*1000 + col into TMEM with tcgen05.st.32x32b (thread = lane,
// register = column), reads it back with tcgen05.ld.16x256b.x2 from lane
// base 0 and 16, prints what every thread of warp 0 received.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2601_11608_b200/csrc/ptx.cuh"
using namespace wfb::ptx;

__global__ void probe(uint32_t* out) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(smem_u32(&tslot), 32);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  // each warp w owns lanes 32w..32w+31; write 16 columns
  uint32_t v[16];
  for (int c = 0; c < 16; ++c) v[c] = (32 * warp + lane) * 1000 + c;
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
               ::"r"(tmem + ((32u * warp) << 16)), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]),
               "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
               "r"(v[15]) : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) {
    for (int lb = 0; lb < 2; ++lb) {
      uint32_t r[8];
      asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(tmem + ((16u * lb) << 16)));
      tmem_ld_wait();
      for (int i = 0; i < 8; ++i) out[(lb * 32 + lane) * 8 + i] = r[i];
    }
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 32); }
}

int main() {
  uint32_t* d; cudaMalloc(&d, 2 * 32 * 8 * 4);
  probe<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  uint32_t h[2 * 32 * 8];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  for (int lb = 0; lb < 2; ++lb)
    for (int t = 0; t < 32; ++t) {
      printf("lanebase %2d thread %2d:", 16 * lb, t);
      for (int i = 0; i < 8; ++i) printf(" %u.%u", h[(lb * 32 + t) * 8 + i] / 1000, h[(lb * 32 + t) * 8 + i] % 1000);
      printf("\n");
    }
  return 0;
}
