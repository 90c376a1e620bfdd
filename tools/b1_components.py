"""Batch-1 (R50 conv1 b1 TF32) per-launch device time in CUDA-graph replay, with the profiling
switches of a PROFILE build: 0x100 no MMA, 0x200 no epilogue, 0x1000 no A loads (needs make PROFILE=1)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2601_11608_b200 as wf  # noqa: E402

x = torch.randn(1, 224, 224, 3, device="cuda")
w = torch.randn(7, 7, 3, 64, device="cuda") * 0.1
b = torch.randn(64, device="cuda")
conv = wf.FoldedConv2d(w, b, x.shape, stride=2, padding=3, dtype=torch.float32)
y = conv(x)
res = {}
flags_list = [int(v, 0) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0]
for fl in flags_list:
    for _ in range(50):
        conv._forward(x, out=y, flags=fl)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g):
            for _ in range(20):
                conv._forward(x, out=y, flags=fl)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(200):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    res[hex(fl)] = e0.elapsed_time(e1) / (200 * 20) * 1e3
print(json.dumps({"graph_us_per_launch": res, "plan": {k: conv.device_plan[k] for k in ("n_tiles", "tile_rows", "wbox", "mma_entries")}}))
