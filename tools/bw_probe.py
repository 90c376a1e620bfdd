"""Measure B200 HBM bandwidth for write-only, read-only and copy traffic (torch kernels)."""
import torch
n = 6 * 1024**3 // 2  # 6 GiB of bf16
a = torch.empty(n, dtype=torch.bfloat16, device="cuda")
b = torch.empty(n, dtype=torch.bfloat16, device="cuda")
a.normal_()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
def t(fn, nbytes, iters=10):
    fn(); torch.cuda.synchronize()
    e0.record()
    for _ in range(iters): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    return nbytes / ms / 1e6
print("write-only (fill_)  GB/s", t(lambda: b.fill_(1.0), n * 2))
print("write-only (zero_)  GB/s", t(lambda: b.zero_(), n * 2))
print("copy (read+write)   GB/s", t(lambda: b.copy_(a), n * 4))
s = torch.empty((), dtype=torch.float32, device="cuda")
print("read-only (amax)    GB/s", t(lambda: torch.amax(a), n * 2))
