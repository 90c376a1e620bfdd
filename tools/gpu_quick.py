"""Quick GPU check of the folded conv vs torch fp32 conv (development aid)."""
import sys, time
import torch
import torch.nn.functional as F
sys.path.insert(0, ".")
from paper_2601_11608_b200 import ops, _abi as A

def ref(x, w, b, s, p, relu):
    y = F.conv2d(x.permute(0, 3, 1, 2).double().cpu(), w.permute(3, 2, 0, 1).double().cpu(), None if b is None else b.double().cpu(), stride=s, padding=p)
    y = y.permute(0, 2, 3, 1)
    return torch.relu(y) if relu else y

def run(name, n, h, w_, c, kh, kw, cout, s, p, dt, relu=False, f=0, gs=0, out_dtype=None, ints=False):
    g = torch.Generator(device="cuda").manual_seed(1234)
    if ints:
        x = torch.randint(-4, 5, (n, h, w_, c), device="cuda", generator=g).to(dt)
        w = torch.randint(-4, 5, (kh, kw, c, cout), device="cuda", generator=g).to(dt)
        b = torch.randint(-4, 5, (cout,), device="cuda", generator=g).float()
    else:
        x = (torch.rand((n, h, w_, c), device="cuda", generator=g) * 2 - 1).to(dt)
        w = ((torch.rand((kh, kw, c, cout), device="cuda", generator=g) * 2 - 1) / (kh * kw * c) ** 0.5).to(dt)
        b = (torch.rand((cout,), device="cuda", generator=g) * 2 - 1)
    ff = ops.prepare_filter(w, b, x.shape, (s, s), (p, p), fold=f, group_size=gs)
    y = ops.conv_folded(x, ff, relu=relu, out_dtype=out_dtype)
    torch.cuda.synchronize()
    yr = ref(x.float(), w.float(), b, s, p, relu)
    err = (y.double().cpu() - yr).abs().max().item()
    rel = err / yr.abs().max().item()
    print(f"{name}: plan f={ff.plan.f} gs={ff.plan.group_size} nt={ff.plan.n_tiles} shape={tuple(y.shape)} maxabs={err:.3e} normrel={rel:.3e}", flush=True)
    return rel

if __name__ == "__main__":
    print(torch.cuda.get_device_name(), flush=True)
    run("int R50 small f32out", 2, 32, 32, 3, 7, 7, 64, 2, 3, torch.bfloat16, out_dtype=torch.float32, ints=True)
    run("R50 small", 2, 32, 32, 3, 7, 7, 64, 2, 3, torch.bfloat16)
    run("VGG small", 2, 32, 32, 3, 3, 3, 64, 1, 1, torch.bfloat16)
    run("MNv2 small relu fp16", 2, 32, 32, 3, 3, 3, 32, 2, 1, torch.float16, relu=True)
    run("R50 tf32", 1, 224, 224, 3, 7, 7, 64, 2, 3, torch.float32)
    run("R50 b4", 4, 224, 224, 3, 7, 7, 64, 2, 3, torch.bfloat16)
    run("VGG b2", 2, 224, 224, 3, 3, 3, 64, 1, 1, torch.bfloat16)
    run("MNv2 b4", 4, 224, 224, 3, 3, 3, 32, 2, 1, torch.float16, relu=True)
    run("zeropad R50 c8", 2, 224, 224, 8, 7, 7, 64, 2, 3, torch.bfloat16)
    # timing R50 b1024
    n = 1024
    x = torch.randn(n, 224, 224, 3, device="cuda").to(torch.bfloat16)
    w = (torch.randn(7, 7, 3, 64, device="cuda") * 0.1).to(torch.bfloat16)
    b = torch.randn(64, device="cuda")
    ff = ops.prepare_filter(w, b, x.shape, (2, 2), (3, 3))
    y = ops.conv_folded(x, ff)
    for _ in range(3): ops.conv_folded(x, ff, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): ops.conv_folded(x, ff, out=y)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    byts = x.numel() * 2 + y.numel() * 2
    print(f"R50 b{n}: {ms:.3f} ms  {n/ms*1e3:.0f} img/s  {byts/ms/1e6:.0f} GB/s  useful {2*ff.plan.useful_macs/ms/1e9:.1f} TF/s", flush=True)
