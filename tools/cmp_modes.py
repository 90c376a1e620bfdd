"""Check the TMA-store epilogue (flag 0x1000) against the default epilogue bit-for-bit."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2601_11608_b200 as wf
for (n, h, w, kh, co, s, p, dt, relu) in [(5, 224, 224, 7, 64, 2, 3, torch.bfloat16, False),
                                           (3, 32, 48, 3, 64, 1, 1, torch.bfloat16, False),
                                           (4, 40, 32, 3, 32, 2, 1, torch.float16, True),
                                           (2, 64, 64, 7, 64, 2, 3, torch.float32, False)]:
    x = torch.randn(n, h, w, 3, device="cuda").to(dt)
    wt = (torch.randn(kh, kh, 3, co, device="cuda") * 0.1).to(dt)
    b = torch.randn(co, device="cuda")
    conv = wf.FoldedConv2d(wt, b, x.shape, stride=s, padding=p, dtype=dt)
    y0 = conv(x, relu=relu)
    for fl in (0x1000, 0x2000):
        y1 = torch.full_like(y0, float("nan"))
        conv._forward(x, relu=relu, out=y1, flags=fl)
        torch.cuda.synchronize()
        print(tuple(x.shape), dt, hex(fl), "identical" if torch.equal(y0, y1) else f"DIFF max {(y0.float()-y1.float()).abs().max().item()}")
