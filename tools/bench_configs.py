"""Per-config measurement of the five BASELINE.json first layers, three kernel
variants each (fold / zero-padded Cin 3->8 / unfolded Cin=3), on one B200.

  python tools/bench_configs.py [--iters 20] [--out gpurun_out/configs.json]

For every (config, variant): images/s, useful and issued TFLOP/s, algorithmic
HBM GB/s, fractions of the measured peaks (MEASURED_PEAKS.json), and the
sampled parity error against the CPU oracle (one image). Timing: CUDA events
on the launching stream around `iters` back-to-back launches after 3 warm-up
launches; inputs are resident in HBM. Batches whose input+output exceed the
126 MB L2 need no flush; the R50 batch-1 config (3.8 MB) is timed with an L2
flush (a 256 MB write) between launches, excluded from the kernel time by
per-launch events.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2601_11608_b200 as wf  # noqa: E402

CONFIGS = {  # name: (N, H, W, C, K, Cout, stride, pad, dtype, relu)  -- BASELINE.json configs[0..4]
    "r50_conv1_b1_tf32": (1, 224, 224, 3, 7, 64, 2, 3, torch.float32, False),
    "vgg16_conv1_1_b256_bf16": (256, 224, 224, 3, 3, 64, 1, 1, torch.bfloat16, False),
    "alexnet_conv1_b512_bf16": (512, 227, 227, 3, 11, 96, 4, 0, torch.bfloat16, False),
    "mnv2_stem_b1024_fp16_relu": (1024, 224, 224, 3, 3, 32, 2, 1, torch.float16, True),
    "r50_conv1_b8192_bf16": (8192, 224, 224, 3, 7, 64, 2, 3, torch.bfloat16, False),
}


def peaks():
    """(HBM GB/s, bf16 TFLOP/s, source): MEASURED_PEAKS.json (driver-written), else the
    B200_PROFILING.md fallback, labelled as such."""
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "MEASURED_PEAKS.json"
    except (OSError, KeyError, ValueError):
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


def oracle():
    from tests.oracle_py import Oracle
    so = os.path.join(ROOT, "oracle", "liboracle.so")
    return Oracle(ctypes.CDLL(so))


def time_conv(conv, x, y, relu, iters, flush):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for _ in range(3):
        conv(x, relu=relu, out=y)
    torch.cuda.synchronize()
    if flush is None:
        e0, e1 = ev[0]
        e0.record()
        for _ in range(iters):
            conv(x, relu=relu, out=y)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters
    tot = 0.0
    for e0, e1 in ev:
        flush.zero_()
        e0.record()
        conv(x, relu=relu, out=y)
        e1.record()
    torch.cuda.synchronize()
    for e0, e1 in ev:
        tot += e0.elapsed_time(e1)
    return tot / iters


def bench_gemm_shapes(iters, hbm):
    """fold_tall_skinny vs cuBLAS over a few (K, N, F) tall-skinny shapes (M = 2^24, bf16)."""
    dev = torch.device("cuda", 0)
    out = {}
    for (K, N, F) in ((3, 64, 8), (4, 64, 4), (8, 64, 2), (8, 128, 2), (16, 64, 1), (3, 32, 8)):
        M = 1 << 24
        g = torch.Generator(device=dev).manual_seed(K * 100 + N)
        a = (torch.rand((M, K), generator=g, device=dev) * 2 - 1).bfloat16()
        b = (torch.rand((K, N), generator=g, device=dev) * 2 - 1).bfloat16()
        c = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
        fold = wf.FoldedConv2d(b.reshape(1, 1, K, N), None, (1, M // F, F, K), fold=F)

        def timed(fn):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(iters):
                fn()
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / iters

        tf = timed(lambda: fold(a.reshape(1, M // F, F, K), bias=False, out=c.reshape(1, M // F, F, N)))
        ref = (a[:4096].double() @ b.double()).float().cpu().numpy()
        err = float(np.max(np.abs(c[:4096].float().cpu().numpy() - ref)) / np.max(np.abs(ref)))
        tc = timed(lambda: torch.matmul(a, b, out=c))
        byts = (M * K + M * N) * 2
        out[f"K{K}_N{N}_F{F}"] = {"fold_ms": tf, "cublas_ms": tc, "fold_speedup_vs_cublas": tc / tf,
                                  "fold_hbm_frac": byts / (tf / 1e3) / 1e9 / hbm, "normwise_rel_err": err}
        print(f"gemm K={K} N={N} F={F}: fold {tf:.3f} ms ({byts / (tf / 1e3) / 1e9 / hbm:.2f} of HBM), "
              f"cuBLAS {tc:.3f} ms, x{tc / tf:.2f}, err {err:.1e}", flush=True)
        del a, b, c, fold
        torch.cuda.empty_cache()
    return out


def bench_gemm(iters, hbm):
    """tall-skinny C = A B (M = 2^24 rows, K = 3, N = 64, bf16)
    three ways -- fold_tall_skinny on the folded tcgen05 kernel (F = 8, one
    M row = 8 GEMM rows), the unfolded variant of the same kernel
    (gemm_as_conv1x1), and cuBLAS (torch.matmul) -- on resident HBM data."""
    dev = torch.device("cuda", 0)
    M, K, N, F = 1 << 24, 3, 64, 8
    g = torch.Generator(device=dev).manual_seed(1008)
    a = (torch.rand((M, K), generator=g, device=dev) * 2 - 1).bfloat16()
    b = (torch.rand((K, N), generator=g, device=dev) * 2 - 1).bfloat16()
    c = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    ref = (a[:4096].double() @ b.double()).float().cpu().numpy()
    bytes_min = (M * K + M * N) * 2
    out = {"shape": {"m": M, "k": K, "n": N, "factor": F, "dtype": "bfloat16"}, "min_bytes": bytes_min}

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters

    fold = wf.FoldedConv2d(b.reshape(1, 1, K, N), None, (1, M // F, F, K), fold=F)
    unf = wf.FoldedConv2d(b.reshape(1, 1, K, N), None, (1, M, 1, K), variant="unfolded")
    for name, fn in (("fold_tall_skinny", lambda: fold(a.reshape(1, M // F, F, K), bias=False, out=c.reshape(1, M // F, F, N))),
                     ("unfolded_conv1x1", lambda: unf(a.reshape(1, M, 1, K), bias=False, out=c.reshape(1, M, 1, N))),
                     ("cublas_matmul", lambda: torch.matmul(a, b, out=c))):
        try:
            ms = timed(fn)
            err = float(np.max(np.abs(c[:4096].float().cpu().numpy() - ref)) / np.max(np.abs(ref)))
            out[name] = {"ms": ms, "rows_per_s": M / (ms / 1e3), "hbm_gbs": bytes_min / (ms / 1e3) / 1e9,
                         "hbm_frac": bytes_min / (ms / 1e3) / 1e9 / hbm, "normwise_rel_err": err}
        except Exception as e:  # report, keep going
            out[name] = {"error": f"{type(e).__name__}: {e}"}
    if "ms" in out["fold_tall_skinny"] and "ms" in out["cublas_matmul"]:
        out["fold_speedup_vs_cublas"] = out["cublas_matmul"]["ms"] / out["fold_tall_skinny"]["ms"]
    if "ms" in out["fold_tall_skinny"] and "ms" in out["unfolded_conv1x1"]:
        out["fold_speedup_vs_unfolded"] = out["unfolded_conv1x1"]["ms"] / out["fold_tall_skinny"]["ms"]
    print("tall_skinny_gemm", json.dumps({k: (round(v["ms"], 4) if isinstance(v, dict) and "ms" in v else v)
                                          for k, v in out.items() if k != "shape"}), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "configs.json"))
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    hbm, tc, peak_src = peaks()
    orc = oracle()
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    results = {}
    for name, (N, H, W, C, K, Co, s, p, dt, relu) in CONFIGS.items():
        if args.only and args.only not in name:
            continue
        g = torch.Generator(device=dev).manual_seed(1001 + list(CONFIGS).index(name))
        x = (torch.rand((N, H, W, C), generator=g, device=dev) * 2 - 1).to(dt)
        w = ((torch.rand((K, K, C, Co), generator=g, device=dev) * 2 - 1) / (K * K * C) ** 0.5).to(dt)
        b = torch.rand(Co, generator=g, device=dev) * 2 - 1
        OH = (H + 2 * p - K) // s + 1
        OW = (W + 2 * p - K) // s + 1
        es = x.element_size()
        useful = 2 * OH * OW * Co * K * K * C
        min_bytes = H * W * C * es + OH * OW * Co * es
        out_dt = dt
        y = torch.empty((N, OH, OW, Co), dtype=out_dt, device=dev)
        ref = orc.conv_padded(x[N // 2:N // 2 + 1].float().cpu().numpy(), w.float().cpu().numpy(),
                              b.cpu().numpy(), s, p, relu)
        res = {"shape": {"n": N, "h": H, "w": W, "c": C, "k": K, "cout": Co, "stride": s, "pad": p,
                         "dtype": str(dt).replace("torch.", ""), "relu": relu},
               "useful_gflop_per_img": useful / 1e9, "min_bytes_per_img": min_bytes,
               "useful_ai_flop_per_byte": useful / min_bytes}
        variants = [("fold", None)]
        if dt != torch.float32:
            variants += [("zeropad_cin8", None), ("unfolded", None)]
        for vname, _ in variants:
            try:
                xin, win = x, w
                if vname == "zeropad_cin8":
                    xin = torch.zeros((N, H, W, 8), dtype=dt, device=dev)
                    xin[..., :C] = x
                    win = torch.zeros((K, K, 8, Co), dtype=dt, device=dev)
                    win[:, :, :C] = w
                conv = wf.FoldedConv2d(win, b, xin.shape, stride=s, padding=p, dtype=dt,
                                       variant="unfolded" if vname == "unfolded" else "fold")
                ms = time_conv(conv, xin, y, relu, args.iters, flush if N * min_bytes < (200 << 20) else None)
                got = y[N // 2:N // 2 + 1].float().cpu().numpy()
                err = float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-30))
                d = conv.device_plan
                img_s = N / (ms / 1e3)
                in_bytes = xin.numel() * es
                bytes_launch = in_bytes + y.numel() * es + conv.packed.numel()
                useful_tf = N * useful / (ms / 1e3) / 1e12
                attain = min(tc, useful / min_bytes * hbm / 1e3)
                res[vname] = {
                    "ms": ms, "images_per_s": img_s, "useful_tflops": useful_tf,
                    "issued_tflops": 2 * d["issued_macs"] / (ms / 1e3) / 1e12,
                    "useful_over_issued": N * useful / 2 / d["issued_macs"],
                    "hbm_gbs": bytes_launch / (ms / 1e3) / 1e9, "hbm_frac": bytes_launch / (ms / 1e3) / 1e9 / hbm,
                    "tensor_roofline_frac": useful_tf / tc, "attainable_roofline_frac": useful_tf / attain,
                    "normwise_rel_err": err, "f": d["f"], "producer": d["producer"],
                    "mma_per_tile": d["mma_entries"]}
                del conv
            except Exception as e:  # report, keep going
                res[vname] = {"error": f"{type(e).__name__}: {e}"}
            if vname == "zeropad_cin8":
                del xin, win
        if "zeropad_cin8" in res and "ms" in res.get("zeropad_cin8", {}) and "ms" in res["fold"]:
            res["fold_speedup_vs_zeropad"] = res["zeropad_cin8"]["ms"] / res["fold"]["ms"]
        if "unfolded" in res and "ms" in res.get("unfolded", {}) and "ms" in res["fold"]:
            res["fold_speedup_vs_unfolded"] = res["unfolded"]["ms"] / res["fold"]["ms"]
        results[name] = res
        print(name, json.dumps({k: (round(v["images_per_s"]) if isinstance(v, dict) and "images_per_s" in v else v)
                                for k, v in res.items() if k not in ("shape",)}), flush=True)
        del x, y
        torch.cuda.empty_cache()
    if not args.only or "gemm" in args.only:
        results["tall_skinny_gemm"] = bench_gemm(args.iters, hbm)
        results["tall_skinny_gemm_shapes"] = bench_gemm_shapes(args.iters, hbm)
    results["_peaks"] = {"hbm_gbs": hbm, "bf16_tflops": tc, "source": peak_src}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(results, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
