"""Energy of the epilogue's output-write paths (tools/probes/store_probe.cu).

  python tools/store_probe.py [GB] [seconds]

Writes a GB-sized buffer (default 13.15: R50 conv1 b8192's bf16 output) back to
back for `seconds` per variant while nvidia-smi samples power.draw.instant and
the SM clock; prints GB/s, W, MHz and mJ per GB."""
import ctypes
import json
import os
import subprocess
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
so = os.path.join(ROOT, "tools", "probes", "libstore_probe.so")
if not os.path.exists(so):
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                    "-o", so, os.path.join(ROOT, "tools", "probes", "store_probe.cu")], check=True)
L = ctypes.CDLL(so)
L.store_probe.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_void_p]
gb = float(sys.argv[1]) if len(sys.argv) > 1 else 13.153337344
secs = float(sys.argv[2]) if len(sys.argv) > 2 else 3.0
nbytes = int(gb * 1e9) // 65536 * 65536
y = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
sms = torch.cuda.get_device_properties(0).multi_processor_count
st = torch.cuda.current_stream().cuda_stream
NAMES = {0: "st.global.v8", 1: "st.global.v4", 2: "TMA bulk store (16 KB chunks)", 3: "st.global.v8 no_allocate evict_first"}
res = {}
for var in (0, 2, 1, 3):
    for _ in range(3):
        assert L.store_probe(var, y.data_ptr(), nbytes, sms, st) == 0
    torch.cuda.synchronize()
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=power.draw.instant,clocks.sm", "--format=csv,noheader,nounits",
                            "-lms", "50"], stdout=subprocess.PIPE, text=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    it = 0
    e0.record()
    while time.time() - t0 < secs:
        for _ in range(5):
            L.store_probe(var, y.data_ptr(), nbytes, sms, st)
        it += 5
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    smi.terminate()
    out = smi.communicate()[0].strip().splitlines()
    vals = [tuple(float(v) for v in ln.split(",")) for ln in out if ln.count(",") == 1 and "N/A" not in ln]
    vals = vals[len(vals) // 4:]
    pw = sorted(v[0] for v in vals)[len(vals) // 2] if vals else float("nan")
    mhz = sorted(v[1] for v in vals)[len(vals) // 2] if vals else float("nan")
    ms = e0.elapsed_time(e1) / it
    gbs = nbytes / (ms / 1e3) / 1e9
    res[NAMES[var]] = {"ms": ms, "GB/s": gbs, "W": pw, "sm_MHz": mhz, "mJ_per_GB": pw * ms / (nbytes / 1e9)}
    print(json.dumps({NAMES[var]: res[NAMES[var]]}), flush=True)
