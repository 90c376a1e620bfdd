// Microbenchmark: the MMA issue path of conv_kernel.cuh in isolation -- the
// schedule table in the kernel-parameter constant bank, one elected lane --
// in variants that change only how each MMA's operands are formed:
//   v0 as the kernel: groups of 8 (uniform constant loads first), rolled tail,
//      a = (a_hi:32 | e.x + a_lo), b = (0x4008:32 | e.y + b_lo), idesc = e.z & ~acc, acc = e.z >> 31
//   v1 v0 with every group predicated (no rolled tail)
//   v2 v0 with acc = 1 and idesc = e.z (no per-MMA flag extraction)
//   v3 v0 with b pre-added (e.y is the final low word)
//   v4 v2 + v3
//   v5 v0 + tcgen05.fence::after_thread_sync per tile (the kernel fences after each stage wait)
//   v6 v0 + two commits per tile (stage empty + accumulator full, as the kernel)
//   v7 v0 with the kernel's A addressing: 3 stages x 2 tiles (stage_bytes, tile_shift)
//   v8 v0 on random bf16 operands (data dependence)
// Table from tools/sched_probe.py (same text format as sched_probe.cu).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../../paper_2601_11608_b200/csrc/ptx.cuh"
using namespace wfb::ptx;

struct Args { int n; uint4 table[64]; };
// the kernel's parameter block is ~7.5 KB (ConvArgs with table[384] + TmaMaps);
// BigArgs puts the same 21 entries at the same place inside one that large,
// and a noise warp reads scattered fields the way the epilogue/producer do
struct BigArgs { int n; int pad[300]; uint4 table[384]; int tail[64]; };

template <int V>
__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ Args a, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar, bar2, bar3;
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) {
    uint32_t v = 0x3c003c00u;
    if (V == 8) {  // random bf16 pairs in [-2, 2)
      uint32_t h = (i + 1) * 2654435761u;
      h ^= h >> 13;
      v = (0x3f80u + (h & 0x7Fu) - 0x40u) | ((0x3f80u + ((h >> 8) & 0x7Fu) - 0x40u) << 16) | ((h & 0x80000000u) >> 16) | (h & 0x80000000u);
    }
    ((uint32_t*)smem)[i] = v;
  }
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
  if (warp == 1) {
    const uint32_t a_hi = (1u << 14) | (128u >> 4);
    const uint32_t b_lo = (V == 3 || V == 4) ? 0u : (base + 96 * 1024) >> 4;
    const bool leader = elect_one();
    const int entries = a.n;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t d_base = tmem + (it & 1) * 256;
      const uint32_t a_lo = (V == 7) ? (base + ((it >> 1) % 3) * 33792 + (it & 1) * 2048) >> 4
                                     : (base + (it & 1) * 32768) >> 4;
      auto issue = [&](const uint4& e) {
        const uint64_t adesc = (static_cast<uint64_t>(a_hi) << 32) | (e.x + a_lo);
        const uint64_t bdesc = (static_cast<uint64_t>(0x4008u) << 32) | (e.y + b_lo);
        if (V == 2 || V == 4) {
          if (leader) mma<0>(d_base + e.w, adesc, bdesc, e.z, 1u);
        } else {
          if (leader) mma<0>(d_base + e.w, adesc, bdesc, e.z & 0x7FFFFFFFu, e.z >> 31);
        }
      };
      if (V == 5) tc_fence_after();
      int i = 0;
      if (V == 1) {
        for (; i < entries; i += 8) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (i + j < entries) issue(a.table[i + j]);
        }
      } else {
        for (; i + 8 <= entries; i += 8) {
#pragma unroll
          for (int j = 0; j < 8; ++j) issue(a.table[i + j]);
        }
        for (; i < entries; ++i) issue(a.table[i]);
      }
      if (V == 6 && leader) {
        if (it & 1) mma_commit(smem_u32(&bar2));
        mma_commit(smem_u32(&bar3));
      }
      if (V == 6) __syncwarp();
    }
    if (leader) mma_commit(smem_u32(&bar));
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
    if (threadIdx.x == 32) out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

__global__ void __launch_bounds__(128, 1) probe_big(const __grid_constant__ BigArgs a, int iters, int noise,
                                                   unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ volatile int sink;
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(smem_u32(&tslot), 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 1) {
    const uint32_t a_hi = (1u << 14) | (128u >> 4);
    const uint32_t b_lo = (base + 96 * 1024) >> 4;
    const bool leader = elect_one();
    const int entries = a.n;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t d_base = tmem + (it & 1) * 256;
      const uint32_t a_lo = (base + (it & 1) * 32768) >> 4;
      auto issue = [&](const uint4& e) {
        const uint64_t adesc = (static_cast<uint64_t>(a_hi) << 32) | (e.x + a_lo);
        const uint64_t bdesc = (static_cast<uint64_t>(0x4008u) << 32) | (e.y + b_lo);
        if (leader) mma<0>(d_base + e.w, adesc, bdesc, e.z & 0x7FFFFFFFu, e.z >> 31);
      };
      int i = 0;
      for (; i + 8 <= entries; i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) issue(a.table[i + j]);
      }
      for (; i < entries; ++i) issue(a.table[i]);
    }
    if (leader) mma_commit(smem_u32(&bar));
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
    if (threadIdx.x == 32) out[blockIdx.x] = clock64() - t0;
    if (threadIdx.x == 32) sink = 1;
  } else if (warp >= 2 && noise) {  // scattered parameter reads (chunk_col / tail fields of the kernel)
    int acc = 0;
    for (int k = 0; k < iters * 8; ++k) {
      acc += a.tail[(k * 7 + threadIdx.x) & 63] + a.pad[(k * 13) % 300] + a.table[64 + (k % 320)].x;
      if (sink) break;
    }
    if (acc == 12345) out[0] = acc;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

double run_big(const BigArgs& a, unsigned long long* d, int iters, int noise) {
  cudaFuncSetAttribute(probe_big, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  probe_big<<<148, 128, 210 * 1024>>>(a, iters, noise, d);
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  std::vector<unsigned long long> h(148);
  cudaMemcpy(h.data(), d, 8 * 148, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (auto v : h) mx = v > mx ? v : mx;
  return (double)mx / iters;
}

template <int V>
double run(const Args& a, unsigned long long* d, int iters) {
  cudaFuncSetAttribute(probe<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  probe<V><<<148, 128, 210 * 1024>>>(a, iters, d);
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  std::vector<unsigned long long> h(148);
  cudaMemcpy(h.data(), d, 8 * 148, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (auto v : h) mx = v > mx ? v : mx;
  return (double)mx / iters;
}

// Kernel-shaped launches (item 1): 320 threads like conv_fold_kernel.
//   K=0 warps 2..9 parked on an mbarrier for the whole launch
//   K=1 + the kernel's per-tile accumulator handshake: the issuer commits to
//       tfull[acc] and waits tempty[acc] (2 buffers); warps 2..9 wait tfull,
//       fence, arrive tempty (the MMA-only kernel's epilogue)
//   K=2 K=1 + the epilogue reads its 32 lanes x 256 columns with tcgen05.ld
template <int K>
__global__ void __launch_bounds__(320, 1) probe_k(const __grid_constant__ Args a, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar_end, tfull[2], tempty[2];
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar_end), 1);
    for (int k = 0; k < 2; ++k) { mbar_init(smem_u32(&tfull[k]), 1); mbar_init(smem_u32(&tempty[k]), 256); }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(smem_u32(&tslot), 512);
  asm volatile("fence.proxy.async.shared::cta;");
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 1) {
    const uint32_t a_hi = (1u << 14) | (128u >> 4);
    const uint32_t b_lo = (base + 96 * 1024) >> 4;
    const bool leader = elect_one();
    const int entries = a.n;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int acc = it & 1;
      if (K >= 1) { mbar_wait(smem_u32(&tempty[acc]), ((it >> 1) & 1) ^ 1); tc_fence_after(); }
      const uint32_t d_base = tmem + acc * 256;
      const uint32_t a_lo = (base + (it & 1) * 32768) >> 4;
      int i = 0;
      for (; i + 8 <= entries; i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint4 e = a.table[i + j];
          const uint64_t adesc = (static_cast<uint64_t>(a_hi) << 32) | (e.x + a_lo);
          const uint64_t bdesc = (static_cast<uint64_t>(0x4008u) << 32) | (e.y + b_lo);
          if (leader) mma<0>(d_base + e.w, adesc, bdesc, e.z & 0x7FFFFFFFu, e.z >> 31);
        }
      }
      for (; i < entries; ++i) {
        const uint4 e = a.table[i];
        const uint64_t adesc = (static_cast<uint64_t>(a_hi) << 32) | (e.x + a_lo);
        const uint64_t bdesc = (static_cast<uint64_t>(0x4008u) << 32) | (e.y + b_lo);
        if (leader) mma<0>(d_base + e.w, adesc, bdesc, e.z & 0x7FFFFFFFu, e.z >> 31);
      }
      if (K >= 1 && leader) mma_commit(smem_u32(&tfull[acc]));
      __syncwarp();
    }
    if (leader) mma_commit(smem_u32(&bar_end));
    __syncwarp();
    mbar_wait(smem_u32(&bar_end), 0);
    if (threadIdx.x == 32) out[blockIdx.x] = clock64() - t0;
  } else if (warp >= 2) {
    if (K == 0) {
      mbar_wait(smem_u32(&bar_end), 0);
    } else {
      const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
      float sink = 0.f;
      for (int it = 0; it < iters; ++it) {
        const int acc = it & 1;
        mbar_wait(smem_u32(&tfull[acc]), (it >> 1) & 1);
        tc_fence_after();
        if (K == 2) {
          uint32_t r[32];
          const uint32_t col = acc * 256 + (warp >= 6 ? 128 : 0);
          for (int c = 0; c < 128; c += 32) {
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                         "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                           "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                           "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                           "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                         : "r"(tmem + lane_base + col + c));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            for (int q = 0; q < 32; ++q) sink += __uint_as_float(r[q]);
          }
        }
        tc_fence_before();
        mbar_arrive(smem_u32(&tempty[acc]));
      }
      if (sink == 1234.5f) out[0] = 0;
    }
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int K>
double run_k(const Args& a, unsigned long long* d, int iters) {
  cudaFuncSetAttribute(probe_k<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  probe_k<K><<<148, 320, 210 * 1024>>>(a, iters, d);
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  std::vector<unsigned long long> h(148);
  cudaMemcpy(h.data(), d, 8 * 148, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (auto v : h) mx = v > mx ? v : mx;
  return (double)mx / iters;
}

int main(int argc, char** argv) {
  FILE* f = fopen(argc > 1 ? argv[1] : "gpurun_out/sched_kpair.txt", "r");
  if (!f) { printf("no table\n"); return 1; }
  Args a{};
  std::vector<Args> av(2);
  unsigned ao, lbo, bo, n, col, acc;
  while (a.n < 64 && fscanf(f, "%u %u %u %u %u %u", &ao, &lbo, &bo, &n, &col, &acc) == 6) {
    const uint32_t n8 = n / 8;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (n8 << 17) | ((128u >> 4) << 24);
    a.table[a.n] = make_uint4((ao >> 4) | ((lbo >> 4) << 16), (bo >> 4) | ((n * 16 >> 4) << 16),
                              idesc | (acc ? 0x80000000u : 0u), col);
    ++a.n;
  }
  fclose(f);
  Args a3 = a;  // v3/v4: B low word final (b_lo pre-added; the probe's B sits at base + 96 KB)
  // (the probe cannot know base on the host: v3/v4 use b_lo = 0, i.e. B at smem address 0 -- same cost)
  unsigned long long* d;
  cudaMalloc(&d, 8 * 148);
  const int iters = 2000;
  printf("%d MMAs per tile\n", a.n);
  printf("v0 as kernel          %8.1f cycles/tile\n", run<0>(a, d, iters));
  printf("v1 predicated groups  %8.1f cycles/tile\n", run<1>(a, d, iters));
  printf("v2 const acc          %8.1f cycles/tile\n", run<2>(a, d, iters));
  printf("v3 b pre-added        %8.1f cycles/tile\n", run<3>(a3, d, iters));
  printf("v4 const acc + b      %8.1f cycles/tile\n", run<4>(a3, d, iters));
  printf("v5 + fence per tile   %8.1f cycles/tile\n", run<5>(a, d, iters));
  printf("v6 + 2 commits/tile   %8.1f cycles/tile\n", run<6>(a, d, iters));
  printf("v7 kernel A addressing%8.1f cycles/tile\n", run<7>(a, d, iters));
  printf("v8 random operands    %8.1f cycles/tile\n", run<8>(a, d, iters));
  static BigArgs big{};
  big.n = a.n;
  for (int i = 0; i < a.n; ++i) big.table[i] = a.table[i];
  for (int i = a.n; i < 384; ++i) big.table[i] = make_uint4(i, i, i, i);
  printf("big param block       %8.1f cycles/tile\n", run_big(big, d, iters, 0));
  printf("big + noise warps     %8.1f cycles/tile\n", run_big(big, d, iters, 1));
  printf("k0 320 thr, parked    %8.1f cycles/tile\n", run_k<0>(a, d, iters));
  printf("k1 + acc handshake    %8.1f cycles/tile\n", run_k<1>(a, d, iters));
  printf("k2 + tcgen05.ld drain %8.1f cycles/tile\n", run_k<2>(a, d, iters));
  return 0;
}
