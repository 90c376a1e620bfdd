"""Long randomised soak of the folded conv on the device (test infrastructure, not part of the suite).

Draws geometries from the same generators as tests/test_gpu_fuzz.py with fresh seeds until the time budget
is spent, each with a random planner knob, and checks every case two ways:
  - integer-valued data: bitwise equal to a float64 conv (exact in the fp32 accumulator);
  - real-valued data: finite, normwise error within the north-star tolerance.
Failures are printed with the case and the device plan; the last line is a JSON summary.

    python tools/fuzz_soak.py --seconds 900 --seed 1000
    python tools/fuzz_soak.py --seconds 300 --threads 8 --plans 96   # concurrent launches over many plans
"""
import argparse
import json
import os
import random
import sys
import time
import zlib

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2601_11608_b200 as wf  # noqa: E402

TDT = {"bf16": torch.bfloat16, "f16": torch.float16, "tf32": torch.float32}
TOL = {"bf16": 1e-2, "f16": 1e-2, "tf32": 1e-3}
KNOBS = [{}, {"WF_KPAIR": "0"}, {"WF_KPAIR": "1"}, {"WF_TPS": "1"}, {"WF_TPS": "2"}, {"WF_MCAST": "1"},
         {"WF_MCAST": "0"}, {"WF_GATHER": "1"}, {"WF_GATHER": "2"}, {"WF_RING": "1"}, {"WF_PLANES": "0"},
         {"WF_NACC": "2"}, {"WF_EPI_PP": "1"}, {"WF_PDL": "0"}, {"WF_CTA_PAIR": "1"}]
args_wide = False  # --wide: also Cout 320-1024 (several N-tiles per plan)
args_unfolded = False  # --unfolded: 30% of the 16-bit cases through the unfolded variant (the zero-pad/im2col baseline)
PLAN_KEYS = ("f", "r", "group_size", "n_tiles", "producer", "kstep_mode", "stage_tiles", "wbox", "cta_pair")


def draw(rng):
    """One case: (n, h, w, c, kh, kw, sh, sw, ph, pw, co, dt, relu, knob, out_dtype)."""
    while True:
        kind = rng.random()
        if kind < 0.6:  # small images, rectangular kernels
            n, h, w = rng.randint(1, 6), rng.randint(4, 80), rng.randint(4, 260)
        elif kind < 0.9:  # many tiles per CTA (ring / barrier phase wrap-around)
            n, h, w = rng.randint(32, 320), rng.randint(6, 48), rng.randint(6, 72)
        elif kind < 0.97:  # ImageNet-sized rows
            n, h, w = rng.randint(1, 3), rng.randint(100, 240), rng.randint(200, 240)
        else:  # very wide rows
            n, h, w = rng.randint(1, 3), rng.randint(4, 24), rng.randint(256, 4096)
        c = rng.choice([1, 2, 3, 3, 3, 4, 6, 8])
        kh, kw = rng.choice([1, 2, 3, 5, 7, 11]), rng.choice([1, 2, 3, 5, 7, 11])
        sh, sw = rng.randint(1, 4), rng.randint(1, 4)
        ph, pw = rng.randint(0, kh // 2), rng.randint(0, kw // 2)
        if (h + 2 * ph - kh) // sh + 1 < 1 or (w + 2 * pw - kw) // sw + 1 < 1:
            continue
        co = rng.choice([32, 64, 96, 128, 160, 192, 256] + ([320, 384, 512, 1024] if args_wide else []))
        dt = rng.choice(["bf16", "f16", "tf32"])
        odt = rng.choice(["f32", "f32", "bf16", "f16"])
        case = (n, h, w, c, kh, kw, sh, sw, ph, pw, co, dt, rng.random() < 0.3, rng.randrange(len(KNOBS)), odt)
        if args_unfolded and dt != "tf32" and rng.random() < 0.3:
            case = case + ("unfolded",)
        return case


def f64_conv(x, w, b, case):
    n, h, wd, c, kh, kw, sh, sw, ph, pw, co, dt, relu, knob, odt = case[:15]
    with torch.backends.cudnn.flags(enabled=False):  # cuDNN's float64 algorithms are not exact for every shape
        y = torch.nn.functional.conv2d(x.double().permute(0, 3, 1, 2), w.double().permute(3, 2, 0, 1), b.double(),
                                       stride=(sh, sw), padding=(ph, pw)).permute(0, 2, 3, 1)
    return torch.relu(y) if relu else y


def run_case(case):
    n, h, w, c, kh, kw, sh, sw, ph, pw, co, dt, relu, knob, odt = case[:15]
    variant = case[15] if len(case) > 15 else "fold"
    saved = {k: os.environ.get(k) for k in KNOBS[knob]}
    os.environ.update(KNOBS[knob])
    try:
        tdt = TDT[dt]
        g = torch.Generator(device="cuda").manual_seed(zlib.crc32(repr(case).encode()))
        xi = torch.randint(-3, 4, (n, h, w, c), generator=g, device="cuda").to(tdt)
        wi = torch.randint(-3, 4, (kh, kw, c, co), generator=g, device="cuda").to(tdt)
        bi = torch.randint(-8, 9, (co,), generator=g, device="cuda").float()
        try:
            conv = wf.FoldedConv2d(wi, bi, xi.shape, stride=(sh, sw), padding=(ph, pw), dtype=tdt, variant=variant)
        except wf.UnsupportedError:
            return "skip", None, None
        plan = {k: conv.device_plan.get(k) for k in PLAN_KEYS}
        y = conv(xi, relu=relu, out_dtype=torch.float32).double()
        ref = f64_conv(xi, wi, bi, case)
        if not torch.equal(y, ref):
            return "fail", plan, f"integer data: {int((y != ref).sum())} of {y.numel()} outputs differ"
        # real-valued data through a fresh pack into the same conv's buffers (same plan), every output type
        xr = (torch.rand((n, h, w, c), generator=g, device="cuda") * 2 - 1).to(tdt)
        wr = ((torch.rand((kh, kw, c, co), generator=g, device="cuda") * 2 - 1) / (kh * kw * c) ** 0.5).to(tdt)
        br = torch.rand((co,), generator=g, device="cuda") * 2 - 1
        conv2 = wf.FoldedConv2d(wr, br, xr.shape, stride=(sh, sw), padding=(ph, pw), dtype=tdt, variant=variant)
        out_t = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}[odt]
        if dt == "tf32" and out_t != torch.float32:
            out_t = torch.float32
        yr = conv2(xr, relu=relu, out_dtype=out_t).double()
        refr = f64_conv(xr, wr, br, case)
        if not torch.isfinite(yr).all():
            return "fail", plan, "real data: non-finite output"
        err = ((yr - refr).abs().max() / refr.abs().max().clamp_min(1e-30)).item()
        tol = TOL[dt] if out_t == torch.float32 else 1e-2
        if err > tol:
            return "fail", plan, f"real data: normwise rel err {err:.3e} > {tol} (out {odt})"
        return "pass", plan, None
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def thread_soak(seconds, seed, n_threads, n_convs):
    """Host threads on their own streams launching a pool of random plans (more than the C-ABI's 64-entry
    schedule cache, so entries are evicted while other threads launch from them); every result must equal
    the one computed up front, bitwise."""
    import threading
    rng = random.Random(seed)
    pool = []
    while len(pool) < n_convs:
        case = draw(rng)
        n, h, w, c, kh, kw, sh, sw, ph, pw, co, dt, relu, knob, odt = case[:15]
        if n * h * w * co > 40_000_000:
            continue
        tdt = TDT[dt]
        g = torch.Generator(device="cuda").manual_seed(zlib.crc32(repr(case).encode()))
        x = torch.randint(-3, 4, (n, h, w, c), generator=g, device="cuda").to(tdt)
        wt = torch.randint(-3, 4, (kh, kw, c, co), generator=g, device="cuda").to(tdt)
        b = torch.randint(-8, 9, (co,), generator=g, device="cuda").float()
        try:
            conv = wf.FoldedConv2d(wt, b, x.shape, stride=(sh, sw), padding=(ph, pw), dtype=tdt)
        except wf.UnsupportedError:
            continue
        pool.append((case, conv, x, conv(x, relu=relu, out_dtype=torch.float32)))
    torch.cuda.synchronize()
    errors, counts = [], [0] * n_threads
    t_end = time.time() + seconds

    def worker(ti):
        r = random.Random(seed * 100 + ti)
        stream = torch.cuda.Stream()
        mine = {}
        try:
            with torch.cuda.stream(stream):
                while time.time() < t_end and not errors:
                    k = r.randrange(len(pool))
                    case, conv, x, ref = pool[k]
                    if k not in mine:  # a private clone: its own workspace (re-pitch plans)
                        mine[k] = conv.with_batch(x.shape[0])
                    y = mine[k](x, relu=case[12], out_dtype=torch.float32)
                    stream.synchronize()
                    if not torch.equal(y, ref):
                        errors.append((ti, case))
                    counts[ti] += 1
        except Exception as e:
            errors.append((ti, repr(e)[:300]))

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(n_threads)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    print(json.dumps({"mode": "threads", "threads": n_threads, "plans": len(pool), "launches": sum(counts),
                      "seconds": seconds, "failures": errors[:10]}), flush=True)
    return 1 if errors else 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=600)
    ap.add_argument("--seed", type=int, default=1000)
    ap.add_argument("--max-cases", type=int, default=10 ** 9)
    ap.add_argument("--trace", action="store_true", help="print every case before running it")
    ap.add_argument("--threads", type=int, default=0, help="thread soak over a pool of plans instead")
    ap.add_argument("--plans", type=int, default=96)
    ap.add_argument("--wide", action="store_true", help="also draw Cout 320-1024")
    ap.add_argument("--unfolded", action="store_true", help="also run the unfolded variant")
    args = ap.parse_args()
    global args_wide, args_unfolded
    args_wide = args.wide
    args_unfolded = args.unfolded
    if args.threads:
        return thread_soak(args.seconds, args.seed, args.threads, args.plans)
    rng = random.Random(args.seed)
    t0 = time.time()
    counts = {"pass": 0, "skip": 0, "fail": 0}
    producers, knobs, failures = {}, {}, []
    i = 0
    while time.time() - t0 < args.seconds and i < args.max_cases:
        case = draw(rng)
        i += 1
        if args.trace:
            print("case", i, case, flush=True)
        try:
            status, plan, msg = run_case(case)
        except Exception as e:  # an error the planner did not classify is a finding too
            status, plan, msg = "fail", None, repr(e)[:300]
        counts[status] += 1
        if plan:
            key = plan["producer"] + ("/unfolded" if len(case) > 15 else "")
            producers[key] = producers.get(key, 0) + 1
            kn = json.dumps(KNOBS[case[13]])
            knobs[kn] = knobs.get(kn, 0) + 1
        if i % 50 == 0:
            import resource
            print(f"progress {i} cases {time.time() - t0:.0f}s rss {resource.getrusage(resource.RUSAGE_SELF).ru_maxrss // 1024} MB "
                  f"cuda {torch.cuda.memory_allocated() >> 20} MB reserved {torch.cuda.memory_reserved() >> 20} MB "
                  f"last {case}", flush=True)
        if status == "fail":
            failures.append({"case": case, "plan": plan, "msg": msg})
            print("FAIL", case, plan, msg, flush=True)
    torch.cuda.synchronize()
    print(json.dumps({"cases": i, "seconds": round(time.time() - t0, 1), "seed": args.seed, **counts,
                      "producers": producers, "knobs": knobs, "failures": failures[:20]}), flush=True)
    return 1 if counts["fail"] else 0


if __name__ == "__main__":
    sys.exit(main())
