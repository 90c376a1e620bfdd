"""Run one configured conv a few times (for ncu capture).
Usage: prof_conv.py CONFIG [n] [f] [gs] [iters] [flags] [variant: fold|unfolded]"""
import sys
import torch
sys.path.insert(0, ".")
import paper_2601_11608_b200 as wf

CFG = {  # n, h, w, c, kh, kw, cout, s, p, dtype, relu
    "r50": (8192, 224, 224, 3, 7, 7, 64, 2, 3, torch.bfloat16, False),
    "vgg": (256, 224, 224, 3, 3, 3, 64, 1, 1, torch.bfloat16, False),
    "mnv2": (1024, 224, 224, 3, 3, 3, 32, 2, 1, torch.float16, True),
    "alex": (512, 227, 227, 3, 11, 11, 96, 4, 0, torch.bfloat16, False),
    "r50zp": (8192, 224, 224, 8, 7, 7, 64, 2, 3, torch.bfloat16, False),
}
name = sys.argv[1]
n, h, w_, c, kh, kw, cout, s, p, dt, relu = CFG[name]
if len(sys.argv) > 2: n = int(sys.argv[2])
f = int(sys.argv[3]) if len(sys.argv) > 3 else 0
gs = int(sys.argv[4]) if len(sys.argv) > 4 else 0
x = torch.randn(n, h, w_, c, device="cuda").to(dt)
w = (torch.randn(kh, kw, c, cout, device="cuda") * 0.1).to(dt)
b = torch.randn(cout, device="cuda")
variant = sys.argv[7] if len(sys.argv) > 7 else "fold"
ff = wf.FoldedConv2d(w, b, x.shape, stride=s, padding=p, fold=f, group_size=gs, variant=variant)
y = ff(x, relu=relu)
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 3
flags = int(sys.argv[6], 0) if len(sys.argv) > 6 else 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
for _ in range(iters):
    ff._forward(x, relu=relu, out=y, flags=flags)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / iters
print(f"{name} flags={flags:#x} n={n} f={ff.device_plan["f"]} gs={ff.device_plan["group_size"]} nt={ff.device_plan["n_tiles"]}: {ms:.3f} ms {n/ms*1e3:.0f} img/s "
      f"{(x.numel()*x.element_size()+y.numel()*y.element_size())/ms/1e6:.0f} GB/s")
