"""AlexNet conv1: the re-pitch pass of chunk k+1 on a second stream while chunk k is convolved
(wf_repitch_input + WF_EPI_PREPITCHED) vs the single call (re-pitch pass, then the conv).
  python tools/alex_pipeline.py [n] [chunk counts, e.g. 2,4,7]"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2601_11608_b200 as wf  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
Ks = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2, 4, 7]
g = torch.Generator(device="cuda").manual_seed(3)
x = (torch.rand((n, 227, 227, 3), generator=g, device="cuda") * 2 - 1).bfloat16()
w = ((torch.rand((11, 11, 3, 96), generator=g, device="cuda") * 2 - 1) / 18).bfloat16()
b = torch.rand(96, generator=g, device="cuda") * 2 - 1
conv = wf.FoldedConv2d(w, b, x.shape, stride=4, padding=0, dtype=torch.bfloat16)
y = conv(x)
ref = y.clone()
main = torch.cuda.current_stream()
side = torch.cuda.Stream()


def timed(fn, iters=30):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(iters):
        fn()
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


res = {"n": n, "single_call_ms": timed(lambda: conv(x, out=y))}
for K in Ks:
    cut = [min(n, (n * k // K + 7) // 8 * 8) for k in range(K)] + [n]  # 16-byte aligned chunk starts
    bounds = [(cut[k], cut[k + 1]) for k in range(K) if cut[k + 1] > cut[k]]
    parts = [(lo, hi, conv.with_batch(hi - lo)) for lo, hi in bounds]
    evs = [torch.cuda.Event() for _ in parts]

    def pipelined():
        side.wait_stream(main)  # the previous iteration's convs are done with the workspaces
        with torch.cuda.stream(side):
            for (lo, hi, c), ev in zip(parts, evs):
                c.core.repitch(x[lo:hi].data_ptr(), c.workspace.data_ptr(), side.cuda_stream)
                ev.record(side)
        for (lo, hi, c), ev in zip(parts, evs):
            main.wait_event(ev)
            c._forward(x[lo:hi], out=y[lo:hi], flags=4)  # WF_EPI_PREPITCHED

    y.zero_()
    pipelined()
    torch.cuda.synchronize()
    same = bool(torch.equal(y, ref))
    res[f"pipelined_K{K}_ms"] = timed(pipelined)
    res[f"pipelined_K{K}_bitwise_equal"] = same
print(json.dumps(res))
