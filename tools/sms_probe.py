"""R50 conv1 b8192 under the power cap with the persistent grid limited to fewer SMs (wf_set_num_sms):
does leaving SMs idle buy clock back? 100 launches per sample, interleaved."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2601_11608_b200 as wf  # noqa: E402
from paper_2601_11608_b200 import _abi as A  # noqa: E402

n = 8192
x = (torch.rand((n, 224, 224, 3), device="cuda") * 2 - 1).bfloat16()
w = ((torch.rand((7, 7, 3, 64), device="cuda") * 2 - 1) / 12).bfloat16()
b = torch.rand(64, device="cuda")
conv = wf.FoldedConv2d(w, b, x.shape, stride=2, padding=3, dtype=torch.bfloat16)
y = conv(x)
res = {}
for rep in range(2):
    for sms in (148, 144, 136, 128, 112):
        A.lib().wf_set_num_sms(sms)
        for _ in range(5):
            conv(x, out=y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(100):
            conv(x, out=y)
        e1.record()
        torch.cuda.synchronize()
        res.setdefault(sms, []).append(round(e0.elapsed_time(e1) / 100, 4))
A.lib().wf_set_num_sms(0)
print(json.dumps({"ms_per_launch_by_grid_sms": res}))
