// param_probe.cu -- launch cost vs kernel-parameter size (the conv kernel's
// ConvArgs + TmaMaps are ~10.6 KB): an empty kernel with 64 B vs 10.6 KB of
// __grid_constant__ parameters, launched with cudaLaunchKernelExC like the
// conv (optionally with programmatic stream serialization).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
//        -o tools/probes/libparam_probe.so tools/probes/param_probe.cu
#include <cuda_runtime.h>

namespace {
struct Small { int v[16]; };
struct Big { int v[10600 / 4]; };

__global__ void k_small(const __grid_constant__ Small s, int* out) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0 && s.v[3] == 12345) out[0] = s.v[0];
}
__global__ void k_big(const __grid_constant__ Big s, int* out) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0 && s.v[2000] == 12345) out[0] = s.v[0];
}
}  // namespace

extern "C" int param_probe_launch(int big, int pdl, int grid, int* out, void* stream) {
  static Small s{};
  static Big b{};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(320);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  if (pdl) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  void* args[2] = {big ? static_cast<void*>(&b) : static_cast<void*>(&s), &out};
  return static_cast<int>(cudaLaunchKernelExC(&cfg, big ? reinterpret_cast<const void*>(&k_big)
                                                        : reinterpret_cast<const void*>(&k_small), args));
}
