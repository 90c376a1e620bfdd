"""Batch-1 latency, piece by piece (R50 conv1 b1, fp32 -> TF32 -> fp32).

Host time per call of each layer of the eager path (no synchronisation inside
the loop; the GPU queue absorbs the launches), and the device time per launch
of back-to-back eager launches and of CUDA-graph replays.
  python tools/host_path_probe.py            (WF_PDL=0 to compare without
                                              programmatic dependent launch)
"""
import ctypes
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_11608_b200 as wf  # noqa: E402
from paper_2601_11608_b200 import _abi as A  # noqa: E402

dev = torch.device("cuda", 0)
x = torch.randn(1, 224, 224, 3, device=dev)
w = torch.randn(7, 7, 3, 64, device=dev) * 0.1
b = torch.randn(64, device=dev)
conv = wf.FoldedConv2d(w, b, x.shape, stride=2, padding=3, dtype=torch.float32)
y = conv(x)
torch.cuda.synchronize()
N = 2000


def host_us(fn, n=N):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t = (time.perf_counter() - t0) / n * 1e6
    torch.cuda.synchronize()
    return t


def dev_us(fn, n=N):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


res = {"pdl": os.environ.get("WF_PDL", "1") != "0"}
res["host_current_stream_obj_us"] = host_us(lambda: torch.cuda.current_stream(dev).cuda_stream)
res["host_raw_stream_us"] = host_us(lambda: torch._C._cuda_getCurrentRawStream(0))
st = torch._C._cuda_getCurrentRawStream(0)
xp, yp, pp, bp = x.data_ptr(), y.data_ptr(), conv.packed.data_ptr(), conv.b_rep.data_ptr()
core = conv.core
res["host_core_forward_us"] = host_us(lambda: core.forward(xp, pp, bp, yp, "f32", True, False, st, 0, 0))
# the C-ABI straight from ctypes (what a reference-side binding would call)
L = A.lib()
desc = A.make_desc(1, 224, 224, 3, 7, 7, 64, 2, 2, 3, 3)
plan = A.plan_fold(desc, 0, 0, A.WF_TF32)
fwd = L.wf_conv_fold_fwd_ws
dref, pref = ctypes.byref(desc), ctypes.byref(plan)
res["host_cabi_ctypes_us"] = host_us(lambda: fwd(xp, None, pp, bp, yp, dref, pref, A.WF_F32, 1, st))
res["host_call_us"] = host_us(lambda: conv(x, out=y))
res["host_torch_fill_us"] = host_us(lambda: y.fill_(0.0))
res["dev_eager_call_us"] = dev_us(lambda: conv(x, out=y))
res["dev_eager_core_us"] = dev_us(lambda: core.forward(xp, pp, bp, yp, "f32", True, False, st, 0, 0))
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    with torch.cuda.graph(g):
        for _ in range(20):
            conv(x, out=y)
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
res["dev_graph_us"] = dev_us(g.replay, 100) / 20
# one isolated launch: host call -> result ready
lat = []
for _ in range(200):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    conv(x, out=y)
    torch.cuda.synchronize()
    lat.append((time.perf_counter() - t0) * 1e6)
lat.sort()
res["isolated_call_to_ready_us_median"] = lat[len(lat) // 2]
# correctness of back-to-back launches against the first result
ref = conv(x).clone()
for _ in range(5):
    conv(x, out=y)
torch.cuda.synchronize()
res["repeat_bitwise_equal"] = bool(torch.equal(ref, y))
print(json.dumps(res))
