"""Can the copy engines re-pitch AlexNet's rows (1362 -> 1392 bytes) fast enough to hide the re-pitch
pass under the conv? cudaMemcpy2DAsync device-to-device timing vs the repitch kernel, and the two
concurrent (copy on a second stream while the conv runs)."""
import ctypes
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2601_11608_b200 as wf  # noqa: E402

cudart = ctypes.CDLL("libcudart.so.12") if True else None
cudart.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                     ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
x = (torch.rand((n, 227, 227, 3), device="cuda") * 2 - 1).bfloat16()
ws = torch.empty(n * 227 * 1392, dtype=torch.uint8, device="cuda")
s2 = torch.cuda.Stream()


def dma(stream):
    r = cudart.cudaMemcpy2DAsync(ws.data_ptr(), 1392, x.data_ptr(), 1362, 1362, n * 227, 3, stream.cuda_stream)
    assert r == 0, r


def timed(fn, stream, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(iters):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


cur = torch.cuda.current_stream()
res = {"n": n, "bytes_moved_GB": 2 * n * 227 * 1362 / 1e9}
res["dma_memcpy2d_ms"] = timed(lambda: dma(cur), cur)
res["dma_GBps_read_plus_write"] = res["bytes_moved_GB"] / res["dma_memcpy2d_ms"] * 1e3
w = ((torch.rand((11, 11, 3, 96), device="cuda") * 2 - 1) / 18).bfloat16()
b = torch.rand(96, device="cuda")
conv = wf.FoldedConv2d(w, b, x.shape, stride=4, padding=0, dtype=torch.bfloat16)
y = conv(x)
res["conv_call_ms"] = timed(lambda: conv(x, out=y), cur)


def both():
    s2.wait_stream(cur)
    dma(s2)
    conv(x, out=y)
    cur.wait_stream(s2)


res["dma_beside_conv_ms"] = timed(both, cur)
print(json.dumps(res))
