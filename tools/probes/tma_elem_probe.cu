// tma_elem_probe.cu -- which element-granular TMA views of an unaligned-pitch
// tensor does the B200 TMA unit accept at run time? (cuTensorMapEncodeTiled
// accepts overlapping strides; the hardware may not.) One view per process:
//   tma_elem_probe <config> ; prints the 16 loaded bf16 words or faults.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tma_elem_probe tma_elem_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void probe(const __grid_constant__ CUtensorMap m, int rank, int c0, int c1, int c2, int c3, unsigned* out,
                      int nbytes) {
  __shared__ alignas(1024) unsigned char buf[4096];
  __shared__ alignas(8) unsigned long long bar;
  const unsigned sbuf = static_cast<unsigned>(__cvta_generic_to_shared(buf));
  const unsigned sbar = static_cast<unsigned>(__cvta_generic_to_shared(&bar));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(sbar));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(sbar), "r"(nbytes));
    if (rank == 2)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(sbuf), "l"(&m), "r"(c0), "r"(c1), "r"(sbar) : "memory");
    else if (rank == 3)
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(sbuf), "l"(&m), "r"(c0), "r"(c1), "r"(c2), "r"(sbar) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                   ::"r"(sbuf), "l"(&m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(sbar) : "memory");
    asm volatile(
        "{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], 0; @!p bra W; }" ::"r"(sbar) : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nbytes / 4; i += blockDim.x) out[i] = reinterpret_cast<unsigned*>(buf)[i];
}

int main(int argc, char** argv) {
  const int cfg = argc > 1 ? atoi(argv[1]) : 0;
  const long long E = 227LL * 227 * 3 * 4;  // 4 images of AlexNet input, bf16
  std::vector<unsigned short> h(E);
  for (long long i = 0; i < E; ++i) h[i] = static_cast<unsigned short>(i & 0xFFFF);
  unsigned short* x;
  unsigned* out;
  cudaMalloc(&x, E * 2);
  cudaMalloc(&out, 4096);
  cudaMemcpy(x, h.data(), E * 2, cudaMemcpyHostToDevice);
  using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                           const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                           CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  Enc enc = reinterpret_cast<Enc>(p);
  CUtensorMap m;
  int rank = 0, c[4] = {0, 0, 0, 0}, nbytes = 0;
  const long long R = 681 * 5;  // a row start that is 2-byte aligned only (element 3405)
  CUresult r = CUDA_ERROR_INVALID_VALUE;
  if (cfg == 0) {  // {E, 2^20, 3} strides {48, 16} box {8, 32, 1}
    cuuint64_t d[3] = {(cuuint64_t)E, 1u << 20, 3}, s[2] = {48, 16};
    cuuint32_t b[3] = {8, 32, 1}, es[3] = {1, 1, 1};
    r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, x, d, s, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    rank = 3; c[0] = (int)R; nbytes = 512;
  } else if (cfg == 1) {  // {E, 64} strides {48} box {8, 32}
    cuuint64_t d[2] = {(cuuint64_t)E, 64}, s[1] = {48};
    cuuint32_t b[2] = {8, 32}, es[2] = {1, 1};
    r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, d, s, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    rank = 2; c[0] = (int)R; nbytes = 512;
  } else if (cfg == 2) {  // {16, E/8, 2^20, 3} strides {16, 48, 16} box {8, 1, 32, 1}: start m in [0, 8]
    cuuint64_t d[4] = {16, (cuuint64_t)(E / 8), 1u << 20, 3}, s[3] = {16, 48, 16};
    cuuint32_t b[4] = {8, 1, 32, 1}, es[4] = {1, 1, 1, 1};
    r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, x, d, s, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    rank = 4; c[0] = (int)(R % 8); c[1] = (int)(R / 8); nbytes = 512;
  } else if (cfg == 3) {  // aligned only: {8, E/8, 2^20} strides {16, 48} box {8, 1, 32}
    cuuint64_t d[3] = {8, (cuuint64_t)(E / 8), 1u << 20}, s[2] = {16, 48};
    cuuint32_t b[3] = {8, 1, 32}, es[3] = {1, 1, 1};
    r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, x, d, s, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    rank = 3; c[1] = (int)(R / 8); nbytes = 512;
  } else if (cfg == 4) {  // 1-D contiguous run from any element: {E} box {256}
    cuuint64_t d[2] = {(cuuint64_t)E, 1}, s[1] = {(cuuint64_t)E * 2};
    cuuint32_t b[2] = {256, 1}, es[2] = {1, 1};
    r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, d, s, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    rank = 2; c[0] = (int)R; nbytes = 512;
  }
  printf("cfg %d encode %d\n", cfg, (int)r);
  if (r != CUDA_SUCCESS) return 1;
  probe<<<1, 128>>>(m, rank, c[0], c[1], c[2], c[3], out, nbytes);
  const cudaError_t e = cudaDeviceSynchronize();
  printf("cfg %d run: %s\n", cfg, cudaGetErrorString(e));
  if (e != cudaSuccess) return 2;
  std::vector<unsigned short> o(nbytes / 2);
  cudaMemcpy(o.data(), out, nbytes, cudaMemcpyDeviceToHost);
  // expected: core column 0 of folded pixels w'' = element R + 24 w'' + (0..7)
  int bad = 0;
  for (int w = 0; w < 32 && cfg != 4; ++w)
    for (int k = 0; k < 8; ++k) bad += o[w * 8 + k] != static_cast<unsigned short>((R + 24 * w + k) & 0xFFFF);
  for (int k = 0; k < 256 && cfg == 4; ++k) bad += o[k] != static_cast<unsigned short>((R + k) & 0xFFFF);
  printf("cfg %d first %u %u %u ... mismatches %d\n", cfg, o[0], o[1], o[8], bad);
  return 0;
}
