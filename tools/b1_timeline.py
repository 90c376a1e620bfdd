"""CTA-0 launch timeline (PROFILE build, switch 0x8000): %globaltimer stamps of each role's
milestones, for R50 conv1 b1 TF32 (or `bf16 N` for a larger bf16 batch), isolated and back to back."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2601_11608_b200 as wf  # noqa: E402

dt = torch.float32 if len(sys.argv) < 2 or sys.argv[1] == "tf32" else torch.bfloat16
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1
x = torch.randn(n, 224, 224, 3, device="cuda").to(dt)
w = (torch.randn(7, 7, 3, 64, device="cuda") * 0.1).to(dt)
b = torch.randn(64, device="cuda")
conv = wf.FoldedConv2d(w, b, x.shape, stride=2, padding=3, dtype=dt)
y = conv(x)
for _ in range(20):
    conv(x, out=y)
torch.cuda.synchronize()
print("--- isolated (synchronised before each launch)", flush=True)
for _ in range(3):
    conv._forward(x, out=y, flags=0x8000)
    torch.cuda.synchronize()
print("--- back to back", flush=True)
for _ in range(4):
    conv._forward(x, out=y, flags=0x8000)
torch.cuda.synchronize()
