"""Multicast 2-CTA N-tile cluster (opt-in WF_MCAST=1 at plan time) vs the single-CTA launch: bitwise
output equality on plans with two N-tiles, then launch times.
Usage: python tools/mc_check.py"""
import os
import sys
import torch
sys.path.insert(0, ".")
import paper_2601_11608_b200 as wf  # noqa: E402

CASES = [  # n, h, w, c, kh, cout, s, p, dtype
    ("alex", 64, 227, 227, 3, 11, 96, 4, 0, torch.bfloat16),
    ("alex-odd", 7, 227, 227, 3, 11, 96, 4, 0, torch.bfloat16),
    ("vgg", 16, 224, 224, 3, 3, 64, 1, 1, torch.bfloat16),
    ("small", 5, 40, 64, 3, 5, 96, 2, 2, torch.float16),
]


def run(conv, x, mc, iters=0):
    os.environ["WF_MCAST"] = "1" if mc else "0"
    y = conv(x)
    torch.cuda.synchronize()
    ms = None
    if iters:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(3):
            conv(x, out=y)
        e0.record()
        for _ in range(iters):
            conv(x, out=y)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
    return y, ms


torch.manual_seed(0)
for name, n, h, w_, c, k, co, s, p, dt in CASES:
    x = torch.randn(n, h, w_, c, device="cuda").to(dt)
    w = (torch.randn(k, k, c, co, device="cuda") * 0.1).to(dt)
    b = torch.randn(co, device="cuda")
    conv = wf.FoldedConv2d(w, b, x.shape, stride=s, padding=p, dtype=dt)
    y0, _ = run(conv, x, False)
    y1, _ = run(conv, x, True)
    print(name, "n_tiles", conv.device_plan["n_tiles"], "identical" if torch.equal(y0, y1) else
          f"DIFF max {(y0.float() - y1.float()).abs().max().item()}", flush=True)
for name, n in (("alex", 1024), ("alex", 2048), ("vgg", 512)):
    h, w_, k, co, s, p = (227, 227, 11, 96, 4, 0) if name == "alex" else (224, 224, 3, 64, 1, 1)
    x = torch.randn(n, h, w_, 3, device="cuda").to(torch.bfloat16)
    w = (torch.randn(k, k, 3, co, device="cuda") * 0.1).to(torch.bfloat16)
    conv = wf.FoldedConv2d(w, torch.randn(co, device="cuda"), x.shape, stride=s, padding=p, dtype=torch.bfloat16)
    for rep in range(2):
        _, m0 = run(conv, x, False, 20)
        _, m1 = run(conv, x, True, 20)
        print(f"{name} n={n}: default {m0:.3f} ms, multicast {m1:.3f} ms ({m0 / m1:.3f}x)", flush=True)
