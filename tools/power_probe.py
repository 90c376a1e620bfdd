"""Power / clock of the R50 conv under each profiling switch (sustained loop).

  python tools/power_probe.py [n] [seconds]

For every flag set, runs the folded conv back to back for `seconds` while
nvidia-smi samples power.draw.instant and clocks.sm every 100 ms; prints ms/launch,
median W and MHz, and mJ per image. Profiling switches (conv_kernel.cuh):
0x100 no MMAs, 0x200 no epilogue, 0x1000 no A loads.
"""
import subprocess
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2601_11608_b200 as wf  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
secs = float(sys.argv[2]) if len(sys.argv) > 2 else 3.0
x = torch.randn(n, 224, 224, 3, device="cuda").to(torch.bfloat16)
w = (torch.randn(7, 7, 3, 64, device="cuda") * 0.1).to(torch.bfloat16)
b = torch.randn(64, device="cuda")
conv = wf.FoldedConv2d(w, b, x.shape, stride=2, padding=3)
y = conv(x)
FLAGS = [int(v, 0) for v in sys.argv[3].split(',')] if len(sys.argv) > 3 else [0, 0x100, 0x200, 0x1000, 0x300]
for flags in FLAGS:
    for _ in range(3):
        conv._forward(x, out=y, flags=max(flags, 0))
    torch.cuda.synchronize()
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=power.draw.instant,clocks.sm", "--format=csv,noheader,nounits",
                            "-lms", "100"], stdout=subprocess.PIPE, text=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    it = 0
    e0.record()
    while time.time() - t0 < secs:
        for _ in range(10):
            if flags == -1:  # write-only stream of the same output bytes (torch fill kernel)
                y.fill_(1.0)
            else:
                conv._forward(x, out=y, flags=flags)
        it += 10
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    smi.terminate()
    out = smi.communicate()[0].strip().splitlines()
    vals = [tuple(float(v) for v in ln.split(",")) for ln in out if ln.count(",") == 1]
    vals = vals[len(vals) // 4:]  # drop the ramp
    pw = sorted(v[0] for v in vals)[len(vals) // 2] if vals else float("nan")
    mhz = sorted(v[1] for v in vals)[len(vals) // 2] if vals else float("nan")
    ms = e0.elapsed_time(e1) / it
    print(f"flags={flags:#07x}: {ms:.3f} ms/launch {n / ms * 1e3:.0f} img/s  power {pw:.0f} W  sm {mhz:.0f} MHz  "
          f"{pw * ms / n:.4f} mJ/img", flush=True)
