"""Launch cost vs kernel-parameter size (tools/probes/param_probe.cu): host us per launch call
and device us per launch back to back, 64 B vs 10.6 KB of parameters, with / without PDL."""
import ctypes
import json
import os
import subprocess
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
so = os.path.join(ROOT, "tools", "probes", "libparam_probe.so")
if not os.path.exists(so):
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                    "-o", so, os.path.join(ROOT, "tools", "probes", "param_probe.cu")], check=True)
L = ctypes.CDLL(so)
L.param_probe_launch.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
out = torch.zeros(4, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
res = {}
for big in (0, 1):
    for pdl in (0, 1):
        for grid in (112, 148):
            f = lambda: L.param_probe_launch(big, pdl, grid, out.data_ptr(), st)  # noqa: E731
            for _ in range(2000):
                f()
            torch.cuda.synchronize()
            n = 5000
            t0 = time.perf_counter()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(n):
                f()
            e1.record()
            host = (time.perf_counter() - t0) / n * 1e6
            torch.cuda.synchronize()
            res[f"params={'10.6KB' if big else '64B'} pdl={pdl} grid={grid}"] = {
                "host_us_per_call": host, "device_us_per_launch": e0.elapsed_time(e1) / n * 1e3}
print(json.dumps(res, indent=1))

# the same empty kernels in a CUDA graph (20 launches per graph): the per-launch floor without host cost
gres = {}
for big in (0, 1):
    for pdl in (0, 1):
        f = lambda: L.param_probe_launch(big, pdl, 112, out.data_ptr(), torch.cuda.current_stream().cuda_stream)  # noqa: E731
        f()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g):
                for _ in range(20):
                    f()
        torch.cuda.current_stream().wait_stream(s)
        for _ in range(50):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        gres[f"graph params={'10.6KB' if big else '64B'} pdl={pdl} grid=112"] = e0.elapsed_time(e1) / 4000 * 1e3
print(json.dumps(gres, indent=1))
