// Microbenchmark: issue one M-tile schedule of the folded conv (the real
// table from wf_schedule_describe, written by tools/sched_probe.py) back to
// back on every SM, no barriers, no loads, no epilogue -- the pure tensor-pipe
// time of the schedule -- and variants that isolate what costs cycles:
//   mode 0 as planned, 1 all A LBOs = 2 KB (adjacent core-column regions),
//   2 all A starts = 0 (same A every MMA), 3 every N = 256, 4 collector::a
//   reuse hint between consecutive MMAs with the same A start.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../../paper_2601_11608_b200/csrc/ptx.cuh"
using namespace wfb::ptx;

struct Ent { uint32_t a_off, lbo, b_off, n, col, acc; };
struct Tab { int n; Ent e[64]; };

__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ Tab t, int mode, int iters,
                                               unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(smem_u32(&tslot), 512);
  asm volatile("fence.proxy.async.shared::cta;");
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  const int wu = __shfl_sync(0xffffffff, warp, 0);
  if (wu == 1) {
    const uint32_t a0 = base, b0 = base + 96 * 1024;
    const bool leader = elect_one();
    __syncwarp();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t dcol = (it & 1) * 256;
      for (int i = 0; i < t.n; ++i) {
        const Ent e = t.e[i];
        const uint32_t n = (mode == 3) ? 256u : e.n;
        const uint32_t lbo = (mode == 1) ? 2048u : e.lbo;
        const uint32_t aoff = (mode == 2) ? 0u : e.a_off;
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((n >> 3) << 17) | ((128u >> 4) << 24);
        const uint64_t ad = desc(a0 + aoff, lbo, 128), bd = desc(b0 + e.b_off, n * 16, 128);
        const uint32_t col = (mode == 3) ? 0u : e.col;
        if (leader) {
          if (mode == 4) {
            const bool same_prev = i > 0 && t.e[i - 1].a_off == e.a_off && t.e[i - 1].lbo == e.lbo;
            const bool same_next = i + 1 < t.n && t.e[i + 1].a_off == e.a_off && t.e[i + 1].lbo == e.lbo;
            const uint32_t coll = same_prev ? (same_next ? 2u : 3u) : (same_next ? 1u : 0u);
            mma_coll<0>(tmem + dcol + col, ad, bd, idesc, e.acc | (it > 0), coll);
          } else {
            mma<0>(tmem + dcol + col, ad, bd, idesc, e.acc | (it > 0));
          }
        }
      }
    }
    if (leader) mma_commit(smem_u32(&bar));
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
    if (threadIdx.x == 32) out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

// The same schedule with every descriptor precomputed into registers before
// the timed loop (fully unrolled): the fastest possible issue of the table.
template <int NE>
__global__ void __launch_bounds__(128, 1) probe_reg(const __grid_constant__ Tab t, int mode, int iters,
                                                   unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar, bar2, bar3;
  const int warp = threadIdx.x >> 5;
  const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    mbar_init(smem_u32(&bar2), 1);
    mbar_init(smem_u32(&bar3), 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(smem_u32(&tslot), 512);
  asm volatile("fence.proxy.async.shared::cta;");
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  const int wu = __shfl_sync(0xffffffff, warp, 0);
  if (wu == 1) {
    const uint32_t a0 = base, b0 = base + 96 * 1024;
    uint64_t ad[NE], bd[NE];
    uint32_t id[NE], col[NE], accf[NE];
#pragma unroll
    for (int i = 0; i < NE; ++i) {
      const Ent e = t.e[i];
      const uint32_t n = (mode == 3) ? 256u : e.n;
      id[i] = (1u << 4) | (1u << 7) | (1u << 10) | ((n >> 3) << 17) | ((128u >> 4) << 24);
      ad[i] = desc(a0 + e.a_off, e.lbo, 128);
      bd[i] = desc(b0 + e.b_off, n * 16, 128);
      col[i] = (mode == 3) ? 0u : e.col;
      accf[i] = e.acc;
    }
    const bool leader = elect_one();
    __syncwarp();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t dcol = (it & 1) * 256;
#pragma unroll
      for (int i = 0; i < NE; ++i) {
        if (mode == 7) {  // accumulate flag from a runtime per-entry value (as the kernel's table carries it)
          if (leader) mma<0>(tmem + dcol + col[i], ad[i], bd[i], id[i], accf[i] | static_cast<uint32_t>(it > 0));
        } else {
          if (leader) mma<0>(tmem + dcol + col[i], ad[i], bd[i], id[i], 1u);
        }
      }
      if (mode == 5 || mode == 6) { if (leader) mma_commit(smem_u32(&bar2)); }  // per-tile commit (nobody waits)
      if (mode == 6 && leader && (it & 1)) mma_commit(smem_u32(&bar3));  // + a per-stage commit
    }
    if (leader) mma_commit(smem_u32(&bar));
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
    if (threadIdx.x == 32) out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main(int argc, char** argv) {
  Tab t{};
  FILE* f = fopen(argc > 1 ? argv[1] : "gpurun_out/sched_table.txt", "r");
  if (!f) { printf("no table\n"); return 1; }
  while (t.n < 64 && fscanf(f, "%u %u %u %u %u %u", &t.e[t.n].a_off, &t.e[t.n].lbo, &t.e[t.n].b_off, &t.e[t.n].n,
                            &t.e[t.n].col, &t.e[t.n].acc) == 6) ++t.n;
  fclose(f);
  unsigned long long* d; cudaMalloc(&d, 8 * 148);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  const int iters = 2000;
  double model = 0;
  for (int i = 0; i < t.n; ++i) model += (t.e[i].n / 2 > 32 + t.e[i].n / 4) ? t.e[i].n / 2 : 32 + t.e[i].n / 4;
  printf("%d MMAs per tile, cost model %.0f cycles/tile\n", t.n, model);
  const char* names[] = {"as planned", "A LBO = 2 KB", "A start = 0", "all N = 256", "collector::a reuse"};
  for (int mode = 0; mode < 5; ++mode) {
    probe<<<148, 128, 210 * 1024>>>(t, mode, iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<unsigned long long> h(148);
    cudaMemcpy(h.data(), d, 8 * 148, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0; for (auto v : h) mx = v > mx ? v : mx;
    printf("mode %d %-20s %8.1f cycles/tile (max over SMs)\n", mode, names[mode], (double)mx / iters);
  }
  if (t.n == 21 || t.n == 28) {
    for (int mode : {0, 3, 5, 6, 7}) {
      if (t.n == 21) {
        cudaFuncSetAttribute(probe_reg<21>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
        probe_reg<21><<<148, 128, 210 * 1024>>>(t, mode, iters, d);
      } else {
        cudaFuncSetAttribute(probe_reg<28>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
        probe_reg<28><<<148, 128, 210 * 1024>>>(t, mode, iters, d);
      }
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      std::vector<unsigned long long> h(148);
      cudaMemcpy(h.data(), d, 8 * 148, cudaMemcpyDeviceToHost);
      unsigned long long mx = 0; for (auto v : h) mx = v > mx ? v : mx;
      const char* nm = mode == 0 ? "as planned" : mode == 3 ? "all N = 256" : mode == 5 ? "+commit/tile" : mode == 6 ? "+commit/tile+stage" : "runtime acc flag";
      printf("registers, mode %d %-20s %8.1f cycles/tile (max over SMs)\n", mode, nm, (double)mx / iters);
    }
  }
  return 0;
}
