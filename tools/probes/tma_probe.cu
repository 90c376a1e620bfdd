// Probe: can cuTensorMapEncodeTiled describe the folded-pixel core-column view
// (d0 = 8 bf16, d1 = folded col w' stride P, d2 = row i stride s*rowpitch,
//  d3 = core column q stride 16 B [non-monotonic], d4 = image n)? And does a
// TMA load through it land the canonical K-major [q][i][w'][8] smem layout?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe_kernel(const __grid_constant__ CUtensorMap tm, uint16_t* out, int bytes, int c1, int c2) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar)), "r"(bytes));
    asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                 :: "r"(smem_u32(smem)), "l"(&tm), "r"(0), "r"(c1), "r"(c2), "r"(0), "r"(0), "r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" :: "r"(smem_u32(&bar)));
  for (int i = threadIdx.x; i < bytes / 2; i += blockDim.x) out[i] = ((uint16_t*)smem)[i];
}

int main() {
  const int N = 2, H = 9, W = 64, C = 3, f = 16, s = 2, b = 1;
  const int Wf = W / f, P = f * C * 2, Q = P / 16;
  std::vector<uint16_t> hx((size_t)N * H * W * C);
  for (size_t i = 0; i < hx.size(); ++i) hx[i] = (uint16_t)(i & 0x7fff) | 1;
  uint16_t* dx; cudaMalloc(&dx, hx.size() * 2);
  cudaMemcpy(dx, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice);
  const int rows = (H - b + s - 1) / s;
  const int WB = 6, NR = 3;
  cuuint64_t gdim[5] = {8, (cuuint64_t)Wf, (cuuint64_t)rows, (cuuint64_t)Q, (cuuint64_t)N};
  cuuint64_t gstr[4] = {(cuuint64_t)P, (cuuint64_t)s * W * C * 2, 16, (cuuint64_t)H * W * C * 2};
  cuuint32_t box[5] = {8, (cuuint32_t)WB, (cuuint32_t)NR, (cuuint32_t)Q, 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUtensorMap tm;
  CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, (void*)(dx + (size_t)b * W * C), gdim, gstr, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode 5d non-monotonic: %d\n", (int)r);
  if (r != CUDA_SUCCESS) return 0;
  const int bytes = Q * NR * WB * 16;
  uint16_t* dout; cudaMalloc(&dout, bytes);
  cudaMemset(dout, 0xff, bytes);
  const int c1 = -1, c2 = -1;  // start folded col -1, row -1: exercise OOB fill
  probe_kernel<<<1, 128, bytes + 1024>>>(tm, dout, bytes, c1, c2);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<uint16_t> ho(bytes / 2);
  cudaMemcpy(ho.data(), dout, bytes, cudaMemcpyDeviceToHost);
  long bad = 0, checked = 0;
  for (int q = 0; q < Q; ++q) for (int i = 0; i < NR; ++i) for (int w = 0; w < WB; ++w) for (int e8 = 0; e8 < 8; ++e8) {
    int fw = c1 + w, ri = c2 + i, ih = s * ri + b;
    uint16_t want = 0;
    if (fw >= 0 && fw < Wf && ri >= 0 && ri < rows && ih < H) want = hx[(((size_t)0 * H + ih) * W) * C + (size_t)fw * f * C + q * 8 + e8];
    uint16_t got = ho[(((size_t)q * NR + i) * WB + w) * 8 + e8];
    ++checked; if (got != want) { if (bad < 5) printf("mismatch q%d i%d w%d e%d got %u want %u\n", q, i, w, e8, got, want); ++bad; }
  }
  printf("checked %ld bad %ld\n", checked, bad);
  return 0;
}
