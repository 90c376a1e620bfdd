"""A slice of the random geometries + knobs of tests/test_gpu_fuzz.py, for compute-sanitizer
(memcheck / synccheck): out-of-bounds global or shared accesses that happen not to change results."""
import os
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2601_11608_b200 as wf  # noqa: E402
from test_gpu_fuzz import CASES2, KNOBS, TDT  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 24
ran = 0
for case in CASES2[:count]:
    n, h, w, c, kh, kw, sh, sw, ph, pw, co, dt, relu, knob = case
    for key in ("WF_KPAIR", "WF_TPS", "WF_MCAST", "WF_GATHER", "WF_RING", "WF_PLANES", "WF_NACC", "WF_EPI_PP", "WF_PDL",
                "WF_CTA_PAIR"):
        os.environ.pop(key, None)
    os.environ.update(KNOBS[knob])
    tdt = TDT[dt]
    x = torch.randint(-3, 4, (n, h, w, c), device="cuda").to(tdt)
    wt = torch.randint(-3, 4, (kh, kw, c, co), device="cuda").to(tdt)
    b = torch.randint(-8, 9, (co,), device="cuda").float()
    try:
        conv = wf.FoldedConv2d(wt, b, x.shape, stride=(sh, sw), padding=(ph, pw), dtype=tdt)
    except wf.UnsupportedError:
        continue
    y = conv(x, relu=relu, out_dtype=torch.float32)
    with torch.backends.cudnn.flags(enabled=False):  # exact float64 reference (cuDNN's is not for every shape)
        ref = torch.nn.functional.conv2d(x.double().permute(0, 3, 1, 2), wt.double().permute(3, 2, 0, 1),
                                         b.double(), stride=(sh, sw), padding=(ph, pw)).permute(0, 2, 3, 1)
    if relu:
        ref = torch.relu(ref)
    assert torch.equal(y.double(), ref), case
    ran += 1
torch.cuda.synchronize()
print(f"sanitize fuzz: {ran} cases ok")
