"""Probe: does cuTensorMapEncodeTiled accept an element-granular row view of an
unaligned-pitch NHWC tensor -- dim0 = every element of the tensor (so a box may
start at any element), dim1 = folded pixel (stride 48 B, overlapping dim0),
dim2 = core column (stride 16 B)? Run on the GPU box; prints the CUresult."""
import ctypes

import torch

cuda = ctypes.CDLL("libcuda.so.1")
cuda.cuInit(0)
x = torch.zeros(512 * 227 * 227 * 3, dtype=torch.bfloat16, device="cuda")
tmap = (ctypes.c_uint8 * 128)()
CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 = 9
E = x.numel()
for dims, strides, box in [
    ([E, 1 << 20, 3], [48, 16], [8, 32, 1]),
    ([E, 1 << 20], [48], [8, 32]),
    ([E, 64], [48], [8, 32]),
    ([8, 1 << 20], [48], [8, 32]),
]:
    r = len(dims)
    gdim = (ctypes.c_uint64 * r)(*dims)
    gstr = (ctypes.c_uint64 * (r - 1))(*strides)
    bdim = (ctypes.c_uint32 * r)(*box)
    estr = (ctypes.c_uint32 * r)(*([1] * r))
    res = cuda.cuTensorMapEncodeTiled(ctypes.byref(tmap), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, r,
                                      ctypes.c_void_p(x.data_ptr()), gdim, gstr, bdim, estr, 0, 0, 2, 0)
    print(dims, strides, box, "->", res)
