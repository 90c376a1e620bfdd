"""Config 1 latency: R50 conv1 batch 1, fp32 in -> TF32 tensor cores -> fp32 out.

Prints, per launch: device time inside a CUDA graph (no host overhead), eager
back-to-back device time (host launch path included when it is the
bottleneck), and the host wall time of one FoldedConv2d.__call__.
"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2601_11608_b200 as wf  # noqa: E402

x = torch.randn(1, 224, 224, 3, device="cuda")
w = torch.randn(7, 7, 3, 64, device="cuda") * 0.1
b = torch.randn(64, device="cuda")
conv = wf.FoldedConv2d(w, b, x.shape, stride=2, padding=3, dtype=torch.float32)
y = conv(x)
for _ in range(20):
    conv(x, out=y)
torch.cuda.synchronize()
N = 200
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    with torch.cuda.graph(g):
        for _ in range(20):
            conv(x, out=y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
g.replay()
e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
graph_us = e0.elapsed_time(e1) / 20 * 1e3
e0.record()
for _ in range(N):
    conv(x, out=y)
e1.record(); torch.cuda.synchronize()
eager_us = e0.elapsed_time(e1) / N * 1e3
t0 = time.perf_counter()
for _ in range(N):
    conv(x, out=y)
host_us = (time.perf_counter() - t0) / N * 1e6
torch.cuda.synchronize()
print(json.dumps({"config": "R50 conv1 b1 224x224 fp32->TF32", "graph_us_per_launch": graph_us,
                  "eager_us_per_launch": eager_us, "host_us_per_call": host_us,
                  "plan": {k: conv.device_plan[k] for k in ("f", "r", "n_tiles", "tile_rows", "wbox")}}))
