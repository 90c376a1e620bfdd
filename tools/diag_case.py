"""Characterise a failing geometry on the device: mismatch counts per batch size and where they sit
(output rows / columns / channels / images). Integer data, exact float64 reference.
    python tools/diag_case.py n h w c kh kw sh sw ph pw cout dtype [ENV=VAL ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2601_11608_b200 as wf  # noqa: E402

TDT = {"bf16": torch.bfloat16, "f16": torch.float16, "tf32": torch.float32}


def run(n, h, w, c, kh, kw, sh, sw, ph, pw, co, dt):
    g = torch.Generator(device="cuda").manual_seed(1)
    tdt = TDT[dt]
    x = torch.randint(-3, 4, (n, h, w, c), generator=g, device="cuda").to(tdt)
    wt = torch.randint(-3, 4, (kh, kw, c, co), generator=g, device="cuda").to(tdt)
    b = torch.randint(-8, 9, (co,), generator=g, device="cuda").float()
    conv = wf.FoldedConv2d(wt, b, x.shape, stride=(sh, sw), padding=(ph, pw), dtype=tdt)
    y = conv(x, out_dtype=torch.float32).double()
    torch.backends.cudnn.enabled = "--cudnn" in sys.argv  # the native float64 conv is exact on integers
    ref = torch.nn.functional.conv2d(x.double().permute(0, 3, 1, 2), wt.double().permute(3, 2, 0, 1), b.double(),
                                     stride=(sh, sw), padding=(ph, pw)).permute(0, 2, 3, 1)
    bad = y != ref
    print(f"n={n}: {int(bad.sum())} of {bad.numel()} differ; plan {conv.device_plan}")
    if bad.any():
        for dim, name in enumerate(["image", "oh", "ow", "co"]):
            idx = bad.nonzero()[:, dim]
            u = torch.unique(idx)
            print(f"   {name}: {u.numel()} distinct, min {int(u.min())} max {int(u.max())}, first {u[:12].tolist()}")
        i = bad.nonzero()[0].tolist()
        print("   first bad", i, float(y[tuple(i)]), float(ref[tuple(i)]))


if __name__ == "__main__":
    a = [v for v in sys.argv[1:] if v != "--cudnn"]
    vals = [int(v) for v in a[:11]]
    dt = a[11]
    for kv in a[12:]:
        k, v = kv.split("=")
        os.environ[k] = v
    for n in sorted({1, 2, vals[0]}):
        run(n, *vals[1:], dt)
