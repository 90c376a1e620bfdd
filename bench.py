"""bench.py -- images/s of the B200-native folded first-layer conv (BASELINE.json metric).

Headline workload (BASELINE.json configs[4], the config the metric is quoted
on for 1/2/4/8 GPUs): ResNet-50 conv1 (7x7, stride 2, pad 3, Cin=3 -> Cout=64),
NHWC 224x224, ONE global batch of 8192 images split into contiguous shards
over the N ranks ("scaling": "strong"), bf16 in / bf16 out, fp32 accumulate,
bias fused, synthetic data (seeded U[-1,1)), random-init weights. Images are
independent, so there is no collective on the hot path. A `weak` sub-record
(8192 images per rank) is measured at N > 1; `--weak` makes it the headline.

A step = one folded tcgen05 conv over the rank's shard. Inputs (2.47 GB / N)
and outputs (13.15 GB / N) exceed the 126 MB L2 at every N <= 8, so no flush
is needed between steps. Timing: W warm-up steps, then K steps bracketed by
barrier + synchronize, CUDA events on the launching stream, max over ranks.

Extra keys: roofline (dominant kernel vs the measured HBM peak), cpu_baseline
(the reference CPU conv2d on rank 0's host cores, every N), e2e (the public
API from pinned host buffers, H2D + D2H inside the timing), variants (fold vs
zero-padded Cin 3->8 vs unfolded Cin=3 of the same kernel), configs (the four
other BASELINE.json configs + configs[4]'s f=16 "Cout=512" expansion, each
with img/s, useful/issued TFLOP/s, both roofline fractions and the reference
CPU path timed in the same run; N=1), verify (first/middle/last image of
every shard vs the CPU oracle), clocks + energy per image.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--weak]

`--gpus N` without a torchrun environment re-launches itself under
`torch.distributed.run` with N ranks; under torchrun WORLD_SIZE must equal N.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "conv1 images/sec & useful TFLOP/s (folded vs zero-pad) at 1/2/4/8 B200"
N_IMG, H, W, C, K, COUT, STRIDE, PAD = 8192, 224, 224, 3, 7, 64, 2, 3
OH = OW = (H + 2 * PAD - K) // STRIDE + 1
USEFUL_FLOP_PER_IMG = 2 * OH * OW * COUT * K * K * C          # 2 x count_macs (src/refconv.cpp:116-122)
IN_BYTES_PER_IMG = H * W * C * 2
OUT_BYTES_PER_IMG = OH * OW * COUT * 2
WORKLOAD = "resnet50_conv1_b8192_224_nhwc_bf16"
VERIFY_TOL = 1e-2  # north star: rel <= 1e-2 for bf16/fp16 vs the reference fp32

# BASELINE.json configs[0..3] + configs[4]'s literal "filter expansion to Cout=512" (f=16, r=8):
# name: (N, H, W, C, K, Cout, stride, pad, dtype name, relu, fold factor (0 = planner's choice))
CONFIGS = {
    "r50_conv1_b1_tf32": (1, 224, 224, 3, 7, 64, 2, 3, "float32", False, 0),
    "vgg16_conv1_1_b256_bf16": (256, 224, 224, 3, 3, 64, 1, 1, "bfloat16", False, 0),
    "alexnet_conv1_b512_bf16": (512, 227, 227, 3, 11, 96, 4, 0, "bfloat16", False, 0),
    "mnv2_stem_b1024_fp16_relu": (1024, 224, 224, 3, 3, 32, 2, 1, "float16", True, 0),
    "r50_conv1_b8192_bf16_f16_cout512": (8192, 224, 224, 3, 7, 64, 2, 3, "bfloat16", False, 16),
}


def load_peaks() -> dict:
    """MEASURED_PEAKS.json (driver-written) else the B200_PROFILING.md fallback, labelled as such."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm_gbs": float(p["hbm_gbs"]), "bf16_tflops": float(p["bf16_tflops"]),
                "bf16_tflops_sustained": float(p.get("bf16_tflops_sustained", p["bf16_tflops"])),
                "src": "MEASURED_PEAKS.json"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1590.0,
                "src": "fallback (B200_PROFILING.md)"}


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


# ------------------------------------------------------------------ CPU side
def _ref_lib():
    """(ctypes lib, kind): the reference compiled here (oracle/_ref), else our C port."""
    ref = os.path.join(ROOT, "oracle", "_ref", "libwidthfold_ref.so")
    if os.path.exists(ref):
        return ctypes.CDLL(ref), "reference"
    port = os.path.join(ROOT, "oracle", "liboracle.so")
    if not os.path.exists(port):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), port], check=True, capture_output=True)
    return ctypes.CDLL(port), "port"


def cpu_conv_images(seconds: float, threads: int, geom=None) -> dict:
    """Reference CPU conv path on host threads for ~`seconds`: per image, the
    VALID conv2d on the explicitly zero-padded input, then bias_add (+ReLU for
    MNv2, which the reference lacks). Threads work on
    independent images. geom = (H, W, C, K, Cout, s, p, relu)."""
    h, w_, c, k, co, s, p, relu = geom or (H, W, C, K, COUT, STRIDE, PAD, False)
    oh, ow = (h + 2 * p - k) // s + 1, (w_ + 2 * p - k) // s + 1
    lib, kind = _ref_lib()
    fp = ctypes.POINTER(ctypes.c_float)
    i64 = ctypes.c_int64
    rng = np.random.default_rng(7)
    xp = np.zeros((1, h + 2 * p, w_ + 2 * p, c), np.float32)
    xp[:, p:p + h, p:p + w_] = rng.uniform(-1, 1, (1, h, w_, c))
    wt = (rng.uniform(-1, 1, (k, k, c, co)) / np.sqrt(k * k * c)).astype(np.float32)
    b = rng.uniform(-1, 1, co).astype(np.float32)
    counts = [0] * threads
    deadline = time.perf_counter() + seconds

    def work(t):
        y = np.empty((1, oh, ow, co), np.float32)
        while time.perf_counter() < deadline or counts[t] == 0:
            if kind == "reference":
                lib.wfref_conv2d(xp.ctypes.data_as(fp), i64(1), i64(h + 2 * p), i64(w_ + 2 * p), i64(c),
                                 wt.ctypes.data_as(fp), i64(k), i64(k), i64(co), i64(s), i64(s),
                                 b.ctypes.data_as(fp), int(relu), y.ctypes.data_as(fp))
            else:
                lib.or_conv2d(xp.ctypes.data_as(fp), i64(1), i64(h + 2 * p), i64(w_ + 2 * p), i64(c),
                              wt.ctypes.data_as(fp), i64(k), i64(k), i64(co), i64(s), i64(s),
                              y.ctypes.data_as(fp))
                lib.or_bias_add(y.ctypes.data_as(fp), i64(y.size), b.ctypes.data_as(fp), i64(co))
                if relu:
                    lib.or_relu(y.ctypes.data_as(fp), i64(y.size))
            counts[t] += 1

    t0 = time.perf_counter()
    ts = [threading.Thread(target=work, args=(i,)) for i in range(threads)]  # ctypes drops the GIL
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    el = time.perf_counter() - t0
    n = sum(counts)
    useful = 2 * oh * ow * co * k * k * c
    return {"value": n / el, "unit": "images/s", "cores": threads, "kind": kind,
            "sample": f"{n} images of {h}x{w_}x{c} (k{k} s{s} p{p} -> {co}, fp32, zero-padded input, "
                      f"conv2d+bias_add{'+relu' if relu else ''}) in {el:.1f} s on {threads} host threads; "
                      f"{n * useful / el / 1e9:.2f} useful GFLOP/s",
            "seconds": el}


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_conv_images(max(0.05, args.ref_step_seconds), threads)
        if i >= args.warmup:
            vals.append(r)
    n = sum(v["value"] * v["seconds"] for v in vals)
    t = sum(v["seconds"] for v in vals)
    value = n / t
    gb = N_IMG * args.gpus if args.weak else N_IMG
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / len(vals),
            "higher_is_better": True, "scaling": "weak" if args.weak else "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "global_batch": gb,
                       "impl": "CPU reference (host cores of rank 0; a bounded sample per step)"},
            "useful_tflops": value * USEFUL_FLOP_PER_IMG / 1e12,
            "cpu_baseline": {"value": value, "unit": "images/s", "cores": threads, "kind": vals[0]["kind"],
                             "sample": vals[-1]["sample"]},
            "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU side
class ClockSampler:
    """nvidia-smi clocks, throttle reasons and board power sampled during the timed region."""

    # power.draw is a ~1 s moving average on current drivers (it smears the idle time
    # before a sub-second timed region into the figure); power.draw.instant is not.
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.proc = None

    def __enter__(self):
        self.power_field = "power.draw"
        try:
            probe = subprocess.run(["nvidia-smi", "-i", self.gpu_id, "--query-gpu=power.draw.instant",
                                    "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10)
            if probe.returncode == 0 and probe.stdout.strip()[:1].isdigit():
                self.power_field = "power.draw.instant"
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", self.gpu_id, f"--query-gpu={self.FIELDS}{self.power_field}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.06)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self) -> dict:
        sm, mx, reasons, pw = [], 0.0, set(), []
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
                pw.append(float(parts[6]))
            except ValueError:
                continue
            for name, v in zip(self.NAMES, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_median": statistics.median(pw) if pw else None,
                "power_field": getattr(self, "power_field", None)}


def _timed(fn, steps, warmup, stream, barrier):
    """ms per call: `warmup` untimed calls, then `steps` calls between CUDA events on `stream`."""
    import torch
    for _ in range(warmup):
        fn()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    barrier()
    return e0.elapsed_time(e1) / steps


def _verify_images(conv, x, y, wt, bias, stride, pad, relu, idxs, orc):
    """max normwise rel error of images `idxs` of y vs the CPU oracle (reference semantics)."""
    errs = []
    for i in idxs:
        ref = orc.conv_padded(x[i:i + 1].float().cpu().numpy(), wt.float().cpu().numpy(),
                              None if bias is None else bias.float().cpu().numpy(), stride, pad, relu)
        got = y[i:i + 1].float().cpu().numpy()
        errs.append(float(np.max(np.abs(got - ref)) / max(float(np.max(np.abs(ref))), 1e-30)))
    return errs


def _oracle():
    from tests.oracle_py import Oracle
    port = os.path.join(ROOT, "oracle", "liboracle.so")
    if not os.path.exists(port):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), port], check=True, capture_output=True)
    return Oracle(ctypes.CDLL(port))


def measure_configs(args, peaks, dev, orc) -> dict:
    """The other BASELINE.json configs (+ configs[4]'s f=16 Cout=512 expansion),
    one at a time on this GPU: fold / zero-pad Cin 3->8 / unfolded Cin=3 of the
    same kernel, with the reference CPU path timed beside each (bounded sample)."""
    import torch
    import paper_2601_11608_b200 as wf
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    threads = os.cpu_count() or 1
    out = {}
    for ci, (name, (n, h, w_, c, k, co, s, p, dtn, relu, fold)) in enumerate(CONFIGS.items()):
        dt = getattr(torch, dtn)
        g = torch.Generator(device=dev)
        g.manual_seed(1001 + ci)
        x = (torch.rand((n, h, w_, c), generator=g, device=dev) * 2 - 1).to(dt)
        wt = ((torch.rand((k, k, c, co), generator=g, device=dev) * 2 - 1) / (k * k * c) ** 0.5).to(dt)
        b = torch.rand(co, generator=g, device=dev) * 2 - 1
        oh, ow = (h + 2 * p - k) // s + 1, (w_ + 2 * p - k) // s + 1
        es = x.element_size()
        useful = 2 * oh * ow * co * k * k * c
        min_bytes = h * w_ * c * es + oh * ow * co * es
        y = torch.empty((n, oh, ow, co), dtype=dt, device=dev)
        small = n * min_bytes < (200 << 20)  # fits L2: flush between launches
        steps = max(5, args.config_steps)
        res = {"shape": {"n": n, "h": h, "w": w_, "c": c, "k": k, "cout": co, "stride": s, "pad": p,
                         "dtype": dtn, "relu": relu, "fold": fold or "auto"},
               "useful_gflop_per_img": useful / 1e9, "min_bytes_per_img": min_bytes,
               "useful_ai_flop_per_byte": useful / min_bytes,
               "l2": "flushed (256 MB write) between launches" if small else "no flush: in+out exceed L2"}
        variants = [("fold", fold)]
        if dt != torch.float32 and not fold:
            variants += [("zeropad_cin8", 0), ("unfolded_cin3", 0)]
        for vname, f in variants:
            try:
                xin, win = x, wt
                if vname == "zeropad_cin8":
                    xin = torch.zeros((n, h, w_, 8), dtype=dt, device=dev)
                    xin[..., :c] = x
                    win = torch.zeros((k, k, 8, co), dtype=dt, device=dev)
                    win[:, :, :c] = wt
                conv = wf.FoldedConv2d(win, b, xin.shape, stride=s, padding=p, dtype=dt, fold=f,
                                       variant="unfolded" if vname == "unfolded_cin3" else "fold")
                vsteps = max(3, steps // 4) if vname == "unfolded_cin3" else steps
                if small:
                    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                           for _ in range(vsteps)]
                    for _ in range(3):
                        conv(xin, relu=relu, out=y)
                    for e0, e1 in evs:
                        flush.zero_()
                        e0.record(stream)
                        conv(xin, relu=relu, out=y)
                        e1.record(stream)
                    torch.cuda.synchronize(dev)
                    ms = sum(e0.elapsed_time(e1) for e0, e1 in evs) / vsteps
                else:
                    ms = _timed(lambda: conv(xin, relu=relu, out=y), vsteps, 3, stream,
                                lambda: torch.cuda.synchronize(dev))
                d = conv.device_plan
                errs = _verify_images(conv, xin, y, win, b, s, p, relu, sorted({0, n // 2, n - 1}), orc)
                bytes_launch = xin.numel() * es + y.numel() * es + conv.packed.numel()
                useful_tf = n * useful / (ms / 1e3) / 1e12
                attain = min(peaks["bf16_tflops"], useful / min_bytes * peaks["hbm_gbs"] / 1e3)
                res[vname] = {
                    "ms": ms, "images_per_s": n / (ms / 1e3), "useful_tflops": useful_tf,
                    "issued_tflops": 2 * d["issued_macs"] / (ms / 1e3) / 1e12,
                    "useful_over_issued": n * useful / 2 / d["issued_macs"],
                    "hbm_gbs": bytes_launch / (ms / 1e3) / 1e9,
                    "hbm_roofline_frac": bytes_launch / (ms / 1e3) / 1e9 / peaks["hbm_gbs"],
                    "tensor_roofline_frac": useful_tf / peaks["bf16_tflops"],
                    "attainable_roofline_frac": useful_tf / attain,
                    "verify_max_rel_err": max(errs), "verify_images": sorted({0, n // 2, n - 1}),
                    "f": d["f"], "r": d["r"], "n_tiles": d["n_tiles"], "producer": d["producer"],
                    "mma_per_tile": d["mma_entries"]}
                del conv
            except Exception as e:  # report, keep going
                res[vname] = {"error": f"{type(e).__name__}: {e}"}
            if vname == "zeropad_cin8":
                del xin, win
            torch.cuda.empty_cache()
        for vname in ("zeropad_cin8", "unfolded_cin3"):
            if "ms" in res.get(vname, {}) and "ms" in res["fold"]:
                res[f"fold_speedup_vs_{vname}"] = res[vname]["ms"] / res["fold"]["ms"]
        if "zeropad_cin8" in res:
            # the best fold/zero-pad ratio an HBM-bound kernel can reach is the byte ratio
            zb = h * w_ * 8 * es + oh * ow * co * es
            res["zeropad_byte_ratio_bound"] = zb / min_bytes
        if dt == torch.float32:  # batch-1 latency: eager and CUDA-graph replay
            try:
                conv = wf.FoldedConv2d(wt, b, x.shape, stride=s, padding=p, dtype=dt)
                res["latency_us"] = _latency(conv, x, y, dev)
                del conv
            except Exception as e:
                res["latency_us"] = {"error": f"{type(e).__name__}: {e}"}
        if not args.no_cpu:
            cpu = cpu_conv_images(args.config_cpu_seconds, threads, (h, w_, c, k, co, s, p, relu))
            cpu.pop("seconds", None)
            res["cpu_reference"] = cpu
            if "ms" in res["fold"]:
                res["fold_speedup_vs_cpu_reference"] = res["fold"]["images_per_s"] / cpu["value"]
        out[name] = res
        del x, y, wt, b
        torch.cuda.empty_cache()
    out["_peaks"] = {"hbm_gbs": peaks["hbm_gbs"], "bf16_tflops": peaks["bf16_tflops"], "source": peaks["src"],
                     "note": "TF32 (config 1) is measured against the bf16 peak; its own peak is about half"}
    return out


def _latency(conv, x, y, dev) -> dict:
    """Per-launch latency of a small conv (warm GPU: 0.2 s of launches first, so
    the SM clock has ramped up): eager back to back (host launch path included;
    consecutive launches overlap prologue and tail through programmatic
    dependent launch), host wall time per call, CUDA-graph replay, and one
    isolated call from the host to the result being ready (median)."""
    import torch
    t_end = time.perf_counter() + 0.2
    while time.perf_counter() < t_end:
        for _ in range(100):
            conv(x, out=y)
        torch.cuda.synchronize(dev)
    n = 2000
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        conv(x, out=y)
    e1.record()
    torch.cuda.synchronize(dev)
    eager = e0.elapsed_time(e1) / n * 1e3
    t0 = time.perf_counter()
    for _ in range(n):
        conv(x, out=y)
    host = (time.perf_counter() - t0) / n * 1e6
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            for _ in range(20):
                conv(x, out=y)
    torch.cuda.current_stream(dev).wait_stream(side)
    for _ in range(10):
        g.replay()
    torch.cuda.synchronize(dev)
    e0.record()
    for _ in range(50):
        g.replay()
    e1.record()
    torch.cuda.synchronize(dev)
    graph = e0.elapsed_time(e1) / (50 * 20) * 1e3
    iso = []
    for _ in range(200):
        t0 = time.perf_counter()
        conv(x, out=y)
        torch.cuda.synchronize(dev)
        iso.append((time.perf_counter() - t0) * 1e6)
    iso.sort()
    return {"eager_us_per_launch": eager, "host_us_per_call": host, "graph_us_per_launch": graph,
            "isolated_call_to_ready_us_median": iso[len(iso) // 2],
            "note": "warm GPU; eager/graph = device time per launch of back-to-back launches"}


def run_gpu(args) -> None:
    import torch
    import torch.distributed as dist

    import paper_2601_11608_b200 as wf
    from paper_2601_11608_b200 import shard

    rank, local, world = shard.dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus} (launch N ranks for N GPUs)")
    # WF_BENCH_SHARE_GPU=1 (launcher check on a box with fewer GPUs than ranks): ranks share the GPUs
    # round-robin and the scalars travel over gloo -- the numbers are then NOT a scaling measurement
    shared = os.environ.get("WF_BENCH_SHARE_GPU") == "1" and world > torch.cuda.device_count()
    local = local % torch.cuda.device_count() if shared else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    coll = "cpu" if shared else dev  # where the (verification / timing) collectives' tensors live
    if world > 1:
        shard.init("gloo" if shared else "nccl")
    if args.weak:   # N_IMG images per rank
        lo, hi = rank * N_IMG, (rank + 1) * N_IMG
        total = N_IMG * world
    else:           # one global batch of N_IMG split across the ranks
        lo, hi = shard.shard_range(N_IMG, rank, world)
        total = N_IMG
    n = hi - lo
    peaks = load_peaks()
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # ---- synthetic inputs, resident in HBM before timing ---------------------------
    g = torch.Generator(device=dev)
    g.manual_seed(1001 + 4)
    g.manual_seed(1001 + 4 + lo)  # the shard's images: a function of their global index only
    x = (torch.rand((n, H, W, C), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
    g.manual_seed(1005)  # identical weights on every rank
    wt = ((torch.rand((K, K, C, COUT), generator=g, device=dev) * 2 - 1) / (K * K * C) ** 0.5).to(torch.bfloat16)
    bias = torch.rand(COUT, generator=g, device=dev) * 2 - 1
    conv = wf.FoldedConv2d(wt, bias, x.shape, stride=STRIDE, padding=PAD, dtype=torch.bfloat16)
    y = torch.empty(conv.output_shape, dtype=torch.bfloat16, device=dev)

    warm = max(3, args.warmup)
    for _ in range(warm):
        conv(x, out=y)
    barrier()
    gpu_id = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(gpu_id) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            conv(x, out=y)
        ev1.record(stream)
        barrier()
    ms_local = ev0.elapsed_time(ev1)
    ms_total = shard.max_over_ranks(ms_local, coll)
    ms_step = ms_total / args.steps
    value = total / (ms_step / 1e3)
    clocks = clk.summary()

    # ---- verification (outside timing): first / middle / last image of every shard vs the CPU oracle
    verify = None
    orc = None
    if not args.no_verify:
        orc = _oracle()
        idxs = sorted({0, n // 2, n - 1}) if n else []
        errs = _verify_images(conv, x, y, wt, bias, STRIDE, PAD, False, idxs, orc)
        per_rank = shard.gather_scalars([float(lo), float(max(errs) if errs else 0.0), float(len(errs))], coll)
        verify = {"images_per_rank": "first, middle, last image of each shard",
                  "max_rel_err": max(r[1] for r in per_rank), "tol": VERIFY_TOL,
                  "images_checked": int(sum(r[2] for r in per_rank)),
                  "ok": all(r[1] <= VERIFY_TOL for r in per_rank)}

    # ---- weak-scaling sub-record (N > 1): 8192 images per rank ------------------------
    weak = None
    if world > 1 and not args.weak and not args.no_weak:
        del y
        xw = (torch.rand((N_IMG, H, W, C), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
        cw = conv.with_batch(N_IMG)
        yw = torch.empty(cw.output_shape, dtype=torch.bfloat16, device=dev)
        wms = shard.max_over_ranks(_timed(lambda: cw(xw, out=yw), args.steps, warm, stream, barrier), coll)
        weak = {"images_per_rank": N_IMG, "global_batch": N_IMG * world, "ms_per_step": wms,
                "value": N_IMG * world / (wms / 1e3), "unit": "images/s"}
        del xw, yw, cw
        torch.cuda.empty_cache()
        y = torch.empty(conv.output_shape, dtype=torch.bfloat16, device=dev)

    # ---- variants of the same kernel: zero-padded Cin 3 -> 8 and unfolded Cin=3 ----
    variants = {}
    if not args.no_variants:
        xz = torch.zeros((n, H, W, 8), dtype=torch.bfloat16, device=dev)
        xz[..., :C] = x
        wz = torch.zeros((K, K, 8, COUT), dtype=torch.bfloat16, device=dev)
        wz[:, :, :C] = wt
        convz = wf.FoldedConv2d(wz, bias, xz.shape, stride=STRIDE, padding=PAD, dtype=torch.bfloat16)
        zms = shard.max_over_ranks(_timed(lambda: convz(xz, out=y), max(5, args.steps // 4), 3, stream, barrier),
                                   coll)
        del xz, wz
        convu = wf.FoldedConv2d(wt, bias, x.shape, stride=STRIDE, padding=PAD, dtype=torch.bfloat16,
                                variant="unfolded")
        ums = shard.max_over_ranks(_timed(lambda: convu(x, out=y), max(3, args.steps // 20), 2, stream, barrier),
                                   coll)
        for name, ms_, c_, inb in (("fold", ms_step, conv, IN_BYTES_PER_IMG),
                                   ("zeropad_cin8", zms, convz, IN_BYTES_PER_IMG * 8 // 3),
                                   ("unfolded_cin3", ums, convu, IN_BYTES_PER_IMG)):
            d = c_.device_plan
            useful_tf = total * USEFUL_FLOP_PER_IMG / (ms_ / 1e3) / 1e12
            variants[name] = {"images_per_s": total / (ms_ / 1e3), "ms_per_step": ms_,
                              "useful_tflops": useful_tf,
                              "issued_tflops": 2 * d["issued_macs"] * world / (ms_ / 1e3) / 1e12,
                              "useful_over_issued": d["useful_macs"] / d["issued_macs"] * (
                                  C / 8 if name.startswith("zero") else 1.0),
                              "hbm_roofline_frac": n * (inb + OUT_BYTES_PER_IMG) / (ms_ / 1e3) / 1e9
                              / peaks["hbm_gbs"],
                              "tensor_roofline_frac": useful_tf / world / peaks["bf16_tflops"],
                              "fold_factor": d["f"], "group_size": d["group_size"], "a_producer": d["producer"]}
        variants["fold_speedup_vs_zeropad"] = zms / ms_step
        variants["fold_speedup_vs_unfolded"] = ums / ms_step
        variants["zeropad_byte_ratio_bound"] = (IN_BYTES_PER_IMG * 8 / 3 + OUT_BYTES_PER_IMG) / (
            IN_BYTES_PER_IMG + OUT_BYTES_PER_IMG)
        variants["unfolded_note"] = (
            "unfolded Cin=3 builds an explicit im2col A tile with transposer warps (6-byte pixels: no TMA im2col "
            "box); it moves the same HBM bytes as the fold but runs at the hbm_roofline_frac shown, bound by its "
            "gather, so fold_speedup_vs_unfolded measures that gather; zeropad_cin8 (TMA, same kernel) is the "
            "hardware-fair baseline")
        del convz, convu
        torch.cuda.empty_cache()

    # ---- e2e: public API from pinned host buffers, H2D + D2H inside the timing -------
    e2e = None
    if not args.no_e2e:
        ne = n  # the rank's whole shard (15.6 GB of pinned host memory at N=1, 1/N of it per rank)
        xh = torch.empty((ne, H, W, C), dtype=torch.bfloat16).pin_memory()
        xh.copy_(x[:ne].cpu())
        yh = torch.empty((ne,) + tuple(conv.output_shape[1:]), dtype=torch.bfloat16).pin_memory()
        conv.run_host(xh, yh, chunk=args.e2e_chunk)
        barrier()
        es = max(1, min(args.steps, args.e2e_steps))
        ems = shard.max_over_ranks(
            _timed(lambda: conv.run_host(xh, yh, chunk=args.e2e_chunk), es, 0, stream, barrier), coll)
        e2e = {"value": ne * world / (ems / 1e3), "unit": "images/s", "h2d_bytes_per_step": xh.numel() * 2 * world,
               "d2h_bytes_per_step": yh.numel() * 2 * world, "ms_per_step": ems, "steps": es,
               "images_per_rank": ne,
               "path": "FoldedConv2d.run_host (pinned host -> H2D -> folded conv -> D2H, chunked on 2 streams)"}
        # the PCIe ceiling of that leg on this box: plain pinned copies of one chunk, each direction alone
        m = min(ne, args.e2e_chunk)
        sync = lambda: torch.cuda.synchronize(dev)  # noqa: E731
        d2h_ms = _timed(lambda: yh[:m].copy_(y[:m], non_blocking=True), 5, 1, stream, sync)
        h2d_ms = _timed(lambda: x[:m].copy_(xh[:m], non_blocking=True), 5, 1, stream, sync)
        d2h_gbs = yh[:m].numel() * 2 / (d2h_ms / 1e3) / 1e9
        h2d_gbs = xh[:m].numel() * 2 / (h2d_ms / 1e3) / 1e9
        floor_ms = yh.numel() * 2 / d2h_gbs / 1e6  # the output's D2H alone at the copy-engine rate
        e2e["pcie"] = {"d2h_gbs": d2h_gbs, "h2d_gbs": h2d_gbs, "d2h_floor_ms": floor_ms,
                       "floor_over_e2e": floor_ms / ems,
                       "note": "pinned-copy rates measured on this box; the e2e step cannot beat its "
                               "output's device-to-host copy"}
        del xh, yh

    # ---- CPU baseline: rank 0, every N (the other ranks wait at the final barrier) --
    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_conv_images(args.cpu_seconds, os.cpu_count() or 1)
        cpu.pop("seconds", None)

    # ---- the other BASELINE configs (N=1 only: one GPU, measured one at a time) -----
    configs = None
    if world == 1 and not args.no_configs:
        del y
        torch.cuda.empty_cache()
        configs = measure_configs(args, peaks, dev, orc or _oracle())

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant (only) kernel ------------------------------------
    alg_bytes = n * (IN_BYTES_PER_IMG + OUT_BYTES_PER_IMG) + conv.packed.numel() + COUT * 4
    kernel_ms = ms_local / args.steps  # rank 0's own launches, events on the launching stream
    achieved = alg_bytes / (kernel_ms / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath)).get(f"{WORKLOAD}_n{n}")
            traffic = tj if tj is None else float(tj)
        except Exception:
            traffic = None
    useful_tf = total * USEFUL_FLOP_PER_IMG / (ms_step / 1e3) / 1e12
    ai = USEFUL_FLOP_PER_IMG / (IN_BYTES_PER_IMG + OUT_BYTES_PER_IMG)
    attainable = min(peaks["bf16_tflops"], ai * peaks["hbm_gbs"] / 1e3)
    energy = None
    if clocks.get("power_w_median"):
        energy = {"mj_per_image": clocks["power_w_median"] * (ms_step / 1e3) / (total / world) * 1e3,
                  "board_power_w_median": clocks["power_w_median"], "note": "rank 0's board power x its step time"}
    line = {
        "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
        "warmup": warm, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak" if args.weak else "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded U[-1,1) inputs, random-init conv1 weights)",
        "config": {"workload": WORKLOAD, "global_batch": total, "per_gpu_batch": n, "image": [H, W, C],
                   "filter": [K, K, C, COUT], "stride": STRIDE, "padding": PAD, "epilogue": "bias",
                   "fold_factor": conv.device_plan["f"], "parallelism": f"batch-shard{world}",
                   **({"shared_gpu": f"{world} ranks on {torch.cuda.device_count()} GPU(s): launcher check, "
                                     "not a scaling measurement"} if shared else {}),
                   "l2": "no flush: per-step input 2.47 GB/N and output 13.15 GB/N exceed the 126 MB L2"},
        "useful_tflops": useful_tf,
        "tensor_roofline_frac": useful_tf / world / peaks["bf16_tflops"],
        "attainable_roofline_frac": useful_tf / world / attainable,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / peaks["hbm_gbs"], "traffic": traffic, "peak_source": peaks["src"],
                     "algorithmic_bytes_per_launch": alg_bytes, "kernel": "conv_fold_kernel<0,bf16>",
                     "kernel_ms": kernel_ms},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": args.steps,
        "gpu_launches_scope": "per rank: one conv_fold_kernel launch per step",
        "weak": weak,
        "variants": variants,
        "configs": configs,
        "clocks": clocks,
        "energy": energy,
        "verify": verify,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_mock(args) -> None:
    """CPU launcher check (no GPU): every rank joins a gloo group, takes a fake
    per-rank time through the same max-over-ranks path, and rank 0 prints one
    JSON line with what each rank saw."""
    import torch.distributed as dist
    from paper_2601_11608_b200 import shard

    rank, local, world = shard.dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if world > 1:
        shard.init("gloo")
    lo, hi = shard.shard_range(N_IMG, rank, world)
    ms = shard.max_over_ranks(1.0 + rank, "cpu")
    seen = shard.gather_scalars([float(rank), float(local), float(world), float(lo), float(hi)], "cpu")
    if rank == 0:
        print(json.dumps({"mock": True, "n_gpus": world, "max_ms": ms,
                          "ranks": [[int(v) for v in r] for r in seen]}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-step-seconds", type=float, default=0.5)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--e2e-chunk", type=int, default=512)
    ap.add_argument("--config-steps", type=int, default=20)
    ap.add_argument("--config-cpu-seconds", type=float, default=2.0)
    ap.add_argument("--weak", action="store_true", help="headline = 8192 images per rank (weak scaling)")
    ap.add_argument("--no-weak", action="store_true", help="skip the weak-scaling sub-record at N > 1")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--mock", action="store_true", help="CPU launcher check over gloo (no GPU work)")
    args = ap.parse_args()
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        # one process per GPU: re-launch under torchrun (the driver launches torchrun itself)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)]
        sys.exit(subprocess.call(cmd + sys.argv[1:]))
    if args.impl == "reference":
        run_reference(args)
    elif args.mock:
        run_mock(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
