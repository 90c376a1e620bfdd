"""bench.py -- images/s of the B200-native folded first-layer conv (BASELINE.json metric).

Workload (BASELINE.json configs[4], the config the metric is quoted on for
1/2/4/8 GPUs): ResNet-50 conv1 (7x7, stride 2, pad 3, Cin=3 -> Cout=64),
NHWC 224x224, batch 8192 per GPU, bf16 in / bf16 out, fp32 accumulate, bias
fused, synthetic data (seeded U[-1,1)), random-init weights. Images are
independent, so ranks take disjoint shards with no collective on the hot
path; by default every rank holds 8192 images ("scaling": "weak", the work
per GPU is fixed as N grows). --strong instead splits ONE global batch of
8192 into contiguous slices (BASELINE.json configs[4] read literally).

A step = one folded tcgen05 conv over the rank's shard; inputs (2.47 GB at
N=1) exceed the 126 MB L2 so no flush is needed between steps. Timing: W
warm-up steps, then K steps bracketed by barrier + synchronize, CUDA events on
the launching stream, max over ranks. Extra keys: roofline (dominant kernel
vs measured HBM peak), cpu_baseline (the reference CPU conv2d on host cores),
e2e (public API from pinned host buffers, H2D + D2H inside the timing),
variants (fold vs zero-padded Cin 3->8 of the same kernel), clocks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
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


def load_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm_gbs": float(p["hbm_gbs"]), "bf16_tflops": float(p["bf16_tflops"]), "src": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "src": "fallback"}


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


def cpu_conv_images(seconds: float, threads: int) -> dict:
    """Reference CPU conv path on host threads for ~`seconds`: per image, the
    VALID conv2d on the explicitly zero-padded input, then bias_add (BASELINE.md
    section 3). Threads work on independent images."""
    lib, kind = _ref_lib()
    fp = ctypes.POINTER(ctypes.c_float)
    i64 = ctypes.c_int64
    rng = np.random.default_rng(7)
    xp = np.zeros((1, H + 2 * PAD, W + 2 * PAD, C), np.float32)
    xp[:, PAD:PAD + H, PAD:PAD + W] = rng.uniform(-1, 1, (1, H, W, C))
    w = (rng.uniform(-1, 1, (K, K, C, COUT)) / np.sqrt(K * K * C)).astype(np.float32)
    b = rng.uniform(-1, 1, COUT).astype(np.float32)
    counts = [0] * threads
    deadline = time.perf_counter() + seconds

    def work(t):
        y = np.empty((1, OH, OW, COUT), np.float32)
        while time.perf_counter() < deadline or counts[t] == 0:
            if kind == "reference":
                lib.wfref_conv2d(xp.ctypes.data_as(fp), i64(1), i64(H + 2 * PAD), i64(W + 2 * PAD), i64(C),
                                 w.ctypes.data_as(fp), i64(K), i64(K), i64(COUT), i64(STRIDE), i64(STRIDE),
                                 b.ctypes.data_as(fp), 0, y.ctypes.data_as(fp))
            else:
                lib.or_conv2d(xp.ctypes.data_as(fp), i64(1), i64(H + 2 * PAD), i64(W + 2 * PAD), i64(C),
                              w.ctypes.data_as(fp), i64(K), i64(K), i64(COUT), i64(STRIDE), i64(STRIDE),
                              y.ctypes.data_as(fp))
                lib.or_bias_add(y.ctypes.data_as(fp), i64(y.size), b.ctypes.data_as(fp), i64(COUT))
            counts[t] += 1

    t0 = time.perf_counter()
    ts = [threading.Thread(target=work, args=(i,)) for i in range(threads)]  # ctypes drops the GIL
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    el = time.perf_counter() - t0
    n = sum(counts)
    return {"value": n / el, "unit": "images/s", "cores": threads, "kind": kind,
            "sample": f"{n} images of {H}x{W}x{C} (R50 conv1, fp32, zero-padded input, conv2d+bias_add) "
                      f"in {el:.1f} s on {threads} host threads; "
                      f"{n * USEFUL_FLOP_PER_IMG / el / 1e9:.2f} useful GFLOP/s",
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
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / len(vals),
            "higher_is_better": True, "scaling": "strong" if args.strong else "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "global_batch": N_IMG if args.strong else N_IMG * args.gpus,
                       "impl": "CPU reference (host cores of rank 0; a bounded sample per step)"},
            "useful_tflops": value * USEFUL_FLOP_PER_IMG / 1e12,
            "cpu_baseline": {"value": value, "unit": "images/s", "cores": threads, "kind": vals[0]["kind"],
                             "sample": vals[-1]["sample"]},
            "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU side
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", self.gpu_id, f"--query-gpu={self.FIELDS}",
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
        sm, mx, reasons = [], 0.0, set()
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(self.NAMES, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def run_gpu(args) -> None:
    import torch
    import torch.distributed as dist

    import paper_2601_11608_b200 as wf
    from paper_2601_11608_b200 import shard

    rank, local, world = shard.dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        shard.init("nccl")
    if args.strong:  # one global batch of N_IMG split across the ranks
        lo, hi = shard.shard_range(N_IMG, rank, world)
    else:            # N_IMG images per rank
        lo, hi = rank * N_IMG, (rank + 1) * N_IMG
    total = hi - lo if world == 1 else (N_IMG if args.strong else N_IMG * world)
    n = hi - lo
    peaks = load_peaks()

    # ---- synthetic inputs, resident in HBM before timing ---------------------------
    g = torch.Generator(device=dev)
    g.manual_seed(1001 + 4 + rank)
    x = (torch.rand((n, H, W, C), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
    g.manual_seed(1005)  # identical weights on every rank
    wt = ((torch.rand((K, K, C, COUT), generator=g, device=dev) * 2 - 1) / (K * K * C) ** 0.5).to(torch.bfloat16)
    bias = torch.rand(COUT, generator=g, device=dev) * 2 - 1
    conv = wf.FoldedConv2d(wt, bias, x.shape, stride=STRIDE, padding=PAD, dtype=torch.bfloat16)
    y = torch.empty(conv.output_shape, dtype=torch.bfloat16, device=dev)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(max(3, args.warmup)):
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
    ms_total = shard.max_over_ranks(ms_local, dev)
    ms_step = ms_total / args.steps
    value = total / (ms_step / 1e3)

    # ---- verification (outside timing): sampled image vs the CPU oracle; NCCL gather --
    verify = None
    if not args.no_verify:
        from tests.oracle_py import Oracle
        port = os.path.join(ROOT, "oracle", "liboracle.so")
        if not os.path.exists(port):
            subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), port], check=True, capture_output=True)
        orc = Oracle(ctypes.CDLL(port))
        i = n // 2
        ref = orc.conv_padded(x[i:i + 1].float().cpu().numpy(), wt.float().cpu().numpy(), bias.cpu().numpy(),
                              STRIDE, PAD)
        got = y[i:i + 1].float().cpu().numpy()
        err = float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
        csum = float(y.sum(dtype=torch.float64).item())  # no 52 GB float64 copy of the output
        verify = shard.gather_scalars([float(lo + i), err, csum], dev)

    # ---- variants of the same kernel: zero-padded Cin 3 -> 8 (f=2) and unfolded Cin=3 ----
    variants = {}
    if not args.no_variants:
        def time_variant(c_, xin, steps):
            for _ in range(3):
                c_(xin, out=y)
            barrier()
            ev0.record(stream)
            for _ in range(steps):
                c_(xin, out=y)
            ev1.record(stream)
            barrier()
            return shard.max_over_ranks(ev0.elapsed_time(ev1), dev) / steps

        xz = torch.zeros((n, H, W, 8), dtype=torch.bfloat16, device=dev)
        xz[..., :C] = x
        wz = torch.zeros((K, K, 8, COUT), dtype=torch.bfloat16, device=dev)
        wz[:, :, :C] = wt
        convz = wf.FoldedConv2d(wz, bias, xz.shape, stride=STRIDE, padding=PAD, dtype=torch.bfloat16)
        zms = time_variant(convz, xz, max(5, args.steps // 4))
        del xz, wz
        convu = wf.FoldedConv2d(wt, bias, x.shape, stride=STRIDE, padding=PAD, dtype=torch.bfloat16,
                                variant="unfolded")
        ums = time_variant(convu, x, max(3, args.steps // 20))
        for name, ms_, c_ in (("fold", ms_step, conv), ("zeropad_cin8", zms, convz), ("unfolded_cin3", ums, convu)):
            d = c_.device_plan
            variants[name] = {"images_per_s": total / (ms_ / 1e3), "ms_per_step": ms_,
                              "useful_tflops": total * USEFUL_FLOP_PER_IMG / (ms_ / 1e3) / 1e12,
                              "issued_tflops": 2 * d["issued_macs"] * world / (ms_ / 1e3) / 1e12,
                              "useful_over_issued": d["useful_macs"] / d["issued_macs"] * (
                                  C / 8 if name.startswith("zero") else 1.0),
                              "fold_factor": d["f"], "group_size": d["group_size"], "a_producer": d["producer"]}
        variants["fold_speedup_vs_zeropad"] = zms / ms_step
        variants["fold_speedup_vs_unfolded"] = ums / ms_step
        del convz, convu

    # ---- e2e: public API from pinned host buffers, H2D + D2H inside the timing -------
    e2e = None
    if not args.no_e2e:
        # one rank pins its whole shard (15.6 GB of host memory); with several
        # ranks per node each pins at most 4096 images so the job stays well
        # inside host RAM (the metric is a rate, the sample is stated)
        ne = n if world == 1 else min(n, 4096)
        xh = torch.empty((ne, H, W, C), dtype=torch.bfloat16).pin_memory()
        xh.copy_(x[:ne].cpu())
        yh = torch.empty((ne,) + tuple(conv.output_shape[1:]), dtype=torch.bfloat16).pin_memory()
        conv.run_host(xh, yh, chunk=args.e2e_chunk)
        barrier()
        es = max(1, min(args.steps, args.e2e_steps))
        ev0.record(stream)
        for _ in range(es):
            conv.run_host(xh, yh, chunk=args.e2e_chunk)
        ev1.record(stream)
        barrier()
        ems = shard.max_over_ranks(ev0.elapsed_time(ev1), dev) / es
        e2e = {"value": ne * world / (ems / 1e3), "unit": "images/s", "h2d_bytes_per_step": xh.numel() * 2 * world,
               "d2h_bytes_per_step": yh.numel() * 2 * world, "ms_per_step": ems, "steps": es,
               "images_per_rank": ne,
               "path": "FoldedConv2d.run_host (pinned host -> H2D -> folded conv -> D2H, chunked on 2 streams)"}
        del xh, yh

    # ---- CPU baseline: rank 0, N=1 only --------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_conv_images(args.cpu_seconds, os.cpu_count() or 1)
        cpu.pop("seconds", None)

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
    line = {
        "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if args.strong else "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded U[-1,1) inputs, random-init conv1 weights)",
        "config": {"workload": WORKLOAD, "global_batch": total, "per_gpu_batch": n, "image": [H, W, C],
                   "filter": [K, K, C, COUT], "stride": STRIDE, "padding": PAD, "epilogue": "bias",
                   "fold_factor": conv.device_plan["f"], "parallelism": f"batch-shard{world}",
                   "l2": "no flush: per-step input 2.47 GB/N and output 13.15 GB/N exceed the 126 MB L2"},
        "useful_tflops": useful_tf,
        "tensor_roofline_frac": useful_tf / peaks["bf16_tflops"],
        "attainable_roofline_frac": useful_tf / attainable,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / peaks["hbm_gbs"], "traffic": traffic, "peak_source": peaks["src"],
                     "algorithmic_bytes_per_launch": alg_bytes, "kernel": "conv_fold_kernel<0,bf16>",
                     "kernel_ms": kernel_ms},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": args.steps,
        "gpu_launches_scope": "per rank: one conv_fold_kernel launch per step",
        "variants": variants,
        "clocks": clk.summary(),
        "verify": verify,
    }
    print(json.dumps(line), flush=True)
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
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--strong", action="store_true", help="split one global batch of 8192 across the ranks")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--no-verify", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
