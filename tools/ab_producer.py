"""A/B of two plan-time environments on one conv config (bench-like timing:
CUDA events over a run of launches after warm-up; outputs compared bitwise).
Usage: ab_producer.py CONFIG N "ENV_A" "ENV_B" [iters]
  e.g. ab_producer.py alex 512 "" "WF_REPITCH=1"
"""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2601_11608_b200 as wf  # noqa: E402

CFG = {  # n, h, w, c, kh, kw, cout, s, p, dtype, relu (tools/prof_conv.py)
    "r50": (8192, 224, 224, 3, 7, 7, 64, 2, 3, torch.bfloat16, False),
    "vgg": (256, 224, 224, 3, 3, 3, 64, 1, 1, torch.bfloat16, False),
    "mnv2": (1024, 224, 224, 3, 3, 3, 32, 2, 1, torch.float16, True),
    "alex": (512, 227, 227, 3, 11, 11, 96, 4, 0, torch.bfloat16, False),
}


def run(env, x, w, b, s, p, relu, iters):
    saved = {}
    for kv in filter(None, env.split(",")):
        k, v = kv.split("=")
        saved[k] = os.environ.get(k)
        os.environ[k] = v
    try:
        conv = wf.FoldedConv2d(w, b, x.shape, stride=s, padding=p)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    y = conv(x, relu=relu)
    for _ in range(3):
        conv(x, relu=relu, out=y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        conv(x, relu=relu, out=y)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters, y, conv.device_plan


if __name__ == "__main__":
    name, n = sys.argv[1], int(sys.argv[2])
    envs = sys.argv[3:5]
    iters = int(sys.argv[5]) if len(sys.argv) > 5 else 50
    _, h, w_, c, kh, kw, cout, s, p, dt, relu = CFG[name]
    torch.manual_seed(0)
    x = torch.randn(n, h, w_, c, device="cuda").to(dt)
    w = (torch.randn(kh, kw, c, cout, device="cuda") * 0.1).to(dt)
    b = torch.randn(cout, device="cuda")
    outs = []
    for rep in range(2):
        for env in envs:
            ms, y, d = run(env, x, w, b, s, p, relu, iters)
            if rep == 0:
                outs.append(y)
            print(f"{name} n={n} env='{env}' producer={d['producer']} tps={d['stage_tiles']} nt={d['n_tiles']}: "
                  f"{ms:.4f} ms  {n / ms * 1e3 / 1e6:.3f} M img/s")
    print("bitwise equal:", torch.equal(outs[0], outs[1]))
