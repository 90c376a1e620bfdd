import sys, torch
sys.path.insert(0, ".")
import paper_2601_11608_b200 as wf
x = torch.randn(1, 224, 224, 3, device="cuda")
w = torch.randn(7, 7, 3, 64, device="cuda") * 0.1
b = torch.randn(64, device="cuda")
conv = wf.FoldedConv2d(w, b, x.shape, stride=2, padding=3, dtype=torch.float32)
y = conv(x)
for _ in range(5):
    conv(x, out=y)
torch.cuda.synchronize()
# CUDA graph of 20 back-to-back launches: device time per launch without host overhead
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    with torch.cuda.graph(g):
        for _ in range(20):
            conv(x, out=y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
print(f"b1 tf32: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per launch inside a CUDA graph (hot L2)")
e0.record()
for _ in range(20):
    conv(x, out=y)
e1.record(); torch.cuda.synchronize()
print(f"b1 tf32: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per launch, eager back to back")
