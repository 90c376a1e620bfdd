"""PCIe ceiling for bench.py's e2e leg: pinned host <-> device copy bandwidth,
one direction at a time and both at once, with 1 or 2 streams per direction.
Usage: python tools/pcie_probe.py [MB]"""
import json
import sys

import torch

mb = int(sys.argv[1]) if len(sys.argv) > 1 else 822
n = mb * 2**20
dev = torch.device("cuda", 0)
h = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(4)]
d = [torch.empty(n, dtype=torch.uint8, device=dev) for _ in range(4)]
ss = [torch.cuda.Stream(dev) for _ in range(4)]


def run(plan, reps=5):
    """plan: list of (stream index, 'h2d' | 'd2h', buffer index); returns GB/s over all bytes."""
    for _ in range(2):
        for si, kind, bi in plan:
            with torch.cuda.stream(ss[si]):
                (d[bi].copy_(h[bi], non_blocking=True) if kind == "h2d" else h[bi].copy_(d[bi], non_blocking=True))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream(dev)
    e0.record(cur)
    for s in ss:
        s.wait_stream(cur)
    for _ in range(reps):
        for si, kind, bi in plan:
            with torch.cuda.stream(ss[si]):
                (d[bi].copy_(h[bi], non_blocking=True) if kind == "h2d" else h[bi].copy_(d[bi], non_blocking=True))
    for s in ss:
        cur.wait_stream(s)
    e1.record(cur)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return reps * len(plan) * n / ms / 1e6


res = {"chunk_mb": mb,
       "h2d_1stream": run([(0, "h2d", 0)]),
       "d2h_1stream": run([(0, "d2h", 0)]),
       "d2h_2streams": run([(0, "d2h", 0), (1, "d2h", 1)]),
       "h2d+d2h_concurrent_total": run([(0, "h2d", 0), (1, "d2h", 1)]),
       "d2h_4streams": run([(0, "d2h", 0), (1, "d2h", 1), (2, "d2h", 2), (3, "d2h", 3)])}
print(json.dumps(res))
