"""Small shapes of every producer / epilogue variant, for compute-sanitizer
(memcheck / racecheck / synccheck). Prints the normwise error vs torch's conv.
Back-to-back launches on one stream exercise programmatic dependent launch."""
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
# producers for unaligned rows (W=31: 186-byte rows): re-pitch pass (default), in-kernel L2 ring
# (WF_RING=1), staged gather (WF_GATHER=1), direct gather (WF_GATHER=2)
PROD_ENV = {"": {}, "ring": {"WF_RING": "1"}, "gather": {"WF_GATHER": "1"}, "direct": {"WF_GATHER": "2"}}
UNALIGNED = [(2, 33, 50, 3, 96, 2, 1, torch.bfloat16, False, "fold"),    # 300-byte rows
             (2, 51, 227, 11, 96, 4, 0, torch.bfloat16, False, "fold")]  # AlexNet rows (1362 bytes)
RUNS = [(k, c, "") for k in ("0", "1") for c in CASES] + \
       [("1", c, pe) for c in UNALIGNED for pe in ("", "ring", "gather", "direct")]
for kp, (n, h, w_, kh, co, s, p, dt, relu, var), pe in RUNS:
    os.environ["WF_KPAIR"] = kp  # both K-step schedules
    for k in ("WF_RING", "WF_GATHER"):
        os.environ.pop(k, None)
    os.environ.update(PROD_ENV[pe])
    x = torch.randn(n, h, w_, 3, device="cuda").to(dt)
    w = (torch.randn(kh, kh, 3, co, device="cuda") * 0.1).to(dt)
    b = torch.randn(co, device="cuda")
    conv = wf.FoldedConv2d(w, b, x.shape, stride=s, padding=p, dtype=dt, variant=var)
    for flags in ((0, 0x4000) if var == "fold" and dt != torch.float32 and not pe else (0,)):
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
        print(f"kpair={kp} {var:9s} {conv.device_plan['producer']:13s} {str(dt):14s} {kh}x{kh}/s{s}/p{p} n={n} "
              f"flags={flags:#x} normwise err {err:.2e}", flush=True)
        assert err < 2e-2
a = torch.randn(3000 * 8, 3, device="cuda").bfloat16()  # tall-skinny GEMM on the folded kernel
bm = torch.randn(3, 64, device="cuda").bfloat16()
c = wf.fold_tall_skinny(a, bm, 8, precision="bf16").float()
ref = a.float() @ bm.float()
assert ((c - ref).abs().max() / ref.abs().max()).item() < 2e-2
torch.cuda.synchronize()
print("sanitize cases ok")
