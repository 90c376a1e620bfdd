"""Small shapes of every producer / epilogue variant, for compute-sanitizer
(memcheck / racecheck / synccheck). Prints the normwise error vs torch's conv."""
import os
import sys
import torch
import torch.nn.functional as F
sys.path.insert(0, ".")
import paper_2601_11608_b200 as wf

CASES = [  # n, h, w, kh, cout, s, p, dtype, relu, variant
    (2, 24, 32, 7, 64, 2, 3, torch.bfloat16, False, "fold"),
    (2, 16, 16, 3, 64, 1, 1, torch.bfloat16, False, "fold"),
    (2, 31, 31, 11, 96, 4, 0, torch.bfloat16, False, "fold"),      # re-pitch + masked tail
    (2, 16, 16, 3, 32, 2, 1, torch.float16, True, "fold"),
    (1, 24, 32, 7, 64, 2, 3, torch.float32, False, "fold"),        # tf32
    (2, 24, 32, 7, 64, 2, 3, torch.bfloat16, False, "unfolded"),   # row producer, im2col
    (2, 31, 31, 11, 96, 4, 0, torch.bfloat16, False, "unfolded"),
]
for kp, (n, h, w_, kh, co, s, p, dt, relu, var) in [(k, c) for k in ("0", "1") for c in CASES]:
    os.environ["WF_KPAIR"] = kp  # both K-step schedules
    x = torch.randn(n, h, w_, 3, device="cuda").to(dt)
    w = (torch.randn(kh, kh, 3, co, device="cuda") * 0.1).to(dt)
    b = torch.randn(co, device="cuda")
    conv = wf.FoldedConv2d(w, b, x.shape, stride=s, padding=p, dtype=dt, variant=var)
    for flags in ((0, 0x4000) if var == "fold" and dt != torch.float32 else (0,)):
        try:
            y = conv._forward(x, relu=relu, flags=flags).float()
        except wf.UnsupportedError as e:  # the row-producer cross-check has a 64-row stage table
            print(f"{var:9s} {str(dt):14s} {kh}x{kh}/s{s}/p{p} flags={flags:#x} skipped: {e}")
            continue
        ref = F.conv2d(x.float().permute(0, 3, 1, 2), w.float().permute(3, 2, 0, 1), b, stride=s, padding=p)
        ref = ref.permute(0, 2, 3, 1)
        if relu:
            ref = ref.clamp_min(0)
        err = ((y - ref).abs().max() / ref.abs().max()).item()
        print(f"kpair={kp} {var:9s} {str(dt):14s} {kh}x{kh}/s{s}/p{p} flags={flags:#x} normwise err {err:.2e}", flush=True)
        assert err < 2e-2
a = torch.randn(3000 * 8, 3, device="cuda").bfloat16()  # tall-skinny GEMM on the folded kernel
bm = torch.randn(3, 64, device="cuda").bfloat16()
c = wf.fold_tall_skinny(a, bm, 8, precision="bf16").float()
ref = a.float() @ bm.float()
assert ((c - ref).abs().max() / ref.abs().max()).item() < 2e-2
torch.cuda.synchronize()
print("sanitize cases ok")
