// Write-bandwidth probe: which store path reaches the highest HBM write rate on B200?
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__global__ void st128(uint4* p, size_t n, uint32_t v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(v, v, v, v);
}
__global__ void st128cs(uint4* p, size_t n, uint32_t v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    asm volatile("st.global.cs.v4.b32 [%0], {%1,%1,%1,%1};" :: "l"(p + i), "r"(v) : "memory");
}
__global__ void st256(uint4* p, size_t n, uint32_t v) {  // n in 32-byte units
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" :: "l"(p + 2 * i), "r"(v) : "memory");
}
__global__ void st256_evict_first(uint4* p, size_t n, uint32_t v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" :: "l"(p + 2 * i), "r"(v) : "memory");
}
// each CTA: fill 32 KB smem once, then bulk-store it repeatedly to consecutive chunks
__global__ void bulk_store(uint8_t* p, size_t nchunks, uint32_t v) {
  extern __shared__ __align__(128) uint8_t sm[];
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = v;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
    int inflight = 0;
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(p + c * 32768), "r"(s), "r"(32768) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (++inflight > 4) asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
int main() {
  const size_t bytes = 8ull << 30;
  uint8_t* p; cudaMalloc(&p, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaFuncSetAttribute(bulk_store, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  auto run = [&](const char* name, auto launch) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-28s %8.1f GB/s  (%s)\n", name, bytes * 5 / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  for (int mult : {2, 4, 8}) {
    printf("grid = %d x SMs\n", mult);
    run("st.global.v4 (128b)", [&] { st128<<<sms * mult, 512>>>((uint4*)p, bytes / 16, 1); });
    run("st.global.cs.v4", [&] { st128cs<<<sms * mult, 512>>>((uint4*)p, bytes / 16, 1); });
    run("st.global.v8 (256b)", [&] { st256<<<sms * mult, 512>>>((uint4*)p, bytes / 32, 1); });
    run("st.v8 no_alloc evict_first", [&] { st256_evict_first<<<sms * mult, 512>>>((uint4*)p, bytes / 32, 1); });
    run("cp.async.bulk 32KB stores", [&] { bulk_store<<<sms * mult / 2, 128, 32768>>>(p, bytes / 32768, 1); });
  }
  run("cudaMemset", [&] { cudaMemsetAsync(p, 1, bytes); });
  return 0;
}
