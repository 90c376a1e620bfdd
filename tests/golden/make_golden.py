"""Generate tests/golden/*.npz from the UNMODIFIED reference implementation.

Runs only in the build container, where /root/reference exists: it imports the
reference's own pybind11 module, compiled from /root/reference/proj by
oracle/Makefile (target `ref` -> oracle/_ref/_core*.so). The fixtures it writes
are small, committed, and are what the CPU and GPU tests compare against on
boxes without /root/reference.

  python tests/golden/make_golden.py        # rewrites tests/golden/*.npz

Contents (all float32 unless noted):
  kats.npz        reference hand known-answer tests and legality/MAC tables
  conv_cases.npz  reference conv2d (+bias_add) on seeded integer and float data,
                  strided, VALID (src/refconv.cpp:34-95)
  appendix_a.npz  the Appendix-A golden pipeline (B=1,H=32,W=64,K=5,F=8,Cout=1)
  configs.npz     the five BASELINE geometries at reduced size: x, w, b and the
                  reference conv2d of the explicitly zero-padded input (+bias,
                  +ReLU for MNv2) -- x/w/b hold bf16/fp16-representable values
                  so tensor-core results can be compared without quantisation
                  noise in the inputs; an integer-valued copy pins exactness.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
import _core as ref  # noqa: E402  (the reference's own module)

# The five BASELINE.json configs: name -> (B, H, W, C, KH, KW, Cout, stride, pad, relu, dtype)
CONFIGS = {
    "r50_b1": (1, 224, 224, 3, 7, 7, 64, 2, 3, False, "f32"),
    "vgg16": (256, 224, 224, 3, 3, 3, 64, 1, 1, False, "bf16"),
    "alexnet": (512, 227, 227, 3, 11, 11, 96, 4, 0, False, "bf16"),
    "mnv2": (1024, 224, 224, 3, 3, 3, 32, 2, 1, True, "f16"),
    "r50_b8192": (8192, 224, 224, 3, 7, 7, 64, 2, 3, False, "bf16"),
}
# reduced sizes used for golden outputs (same filter geometry, small images)
SMALL = {"r50_b1": (1, 64, 64), "vgg16": (2, 32, 32), "alexnet": (2, 67, 67), "mnv2": (2, 32, 32),
         "r50_b8192": (2, 48, 48)}


def quantize(a: np.ndarray, dtype: str) -> np.ndarray:
    """Round fp32 values to bf16/fp16 and back (device-representable inputs)."""
    if dtype == "f16":
        return a.astype(np.float16).astype(np.float32)
    if dtype == "bf16":
        u = a.astype(np.float32).view(np.uint32).astype(np.uint64)
        u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16  # round-to-nearest-even
        return u.astype(np.uint32).view(np.float32)
    return a.astype(np.float32)


def ref_conv(x, w, b, stride, pad, relu):
    xp = np.pad(x, ((0, 0), (pad, pad), (pad, pad), (0, 0)))
    y = ref.conv2d(xp, w, stride, stride)
    if b is not None:
        y = ref.bias_add(y, b)
    if relu:
        y = np.where(y < 0, np.float32(0), y).astype(np.float32)
    return y


def make_kats():
    out = {}
    out["fold_4"] = ref.fold_input(np.array([10, 11, 12, 13], np.float32).reshape(1, 1, 4, 1), 2)
    x = np.arange(1, 5, dtype=np.float32).reshape(1, 1, 2, 2)
    out["fold_general_in"] = x
    out["fold_general_out"] = ref.fold_input_general(x, 2)
    w = np.array([5, 7], np.float32).reshape(1, 1, 1, 2)
    out["expand_in"] = w
    out["expand_out"] = ref.expand_filter(w, 2)
    out["replicate"] = ref.replicate_bias(np.array([1, 2], np.float32), 3)
    rng = np.random.default_rng(7)
    wg = rng.integers(-4, 5, size=(3, 1, 3, 4)).astype(np.float32)
    out["expand_general_in"] = wg
    out["expand_general_out_f4"] = ref.expand_filter_general(wg, 4)
    # legality / MAC tables
    rows = []
    for shape, filt, f in [([1, 32, 64, 1], [5, 1, 1, 1], 8), ([1, 4, 7, 1], [3, 1, 1, 1], 8),
                           ([1, 16, 16, 3], [3, 3, 3, 4], 2), ([1, 16, 16, 3], [3, 1, 3, 4], 8),
                           ([1, 224, 224, 3], [7, 7, 3, 64], 8), ([1, 227, 227, 3], [11, 11, 3, 96], 8),
                           ([1, 224, 224, 3], [3, 3, 3, 32], 8)]:
        p = ref.check_legality(shape, filt, f)
        rows.append((shape, filt, f, p["status"], p["reason"], p["folded_input_shape"], p["expanded_filter_shape"]))
    out["legality"] = np.array([repr(r) for r in rows])
    rows = []
    for shape, filt in [([1, 16, 16, 3], [3, 1, 3, 4]), ([1, 224, 224, 3], [7, 7, 3, 64]),
                        ([1, 227, 227, 3], [11, 11, 3, 96]), ([1, 16, 16, 8], [3, 1, 8, 4]),
                        ([1, 6, 6, 3], [1, 1, 3, 2])]:
        p = ref.choose_fold_factor(shape, filt)
        rows.append((shape, filt, p["status"], p["reason"], p["factor"], p["folded_input_shape"],
                     p["expanded_filter_shape"]))
    out["choose"] = np.array([repr(r) for r in rows])
    mr = ref.mac_report([1, 32, 64, 1], [5, 1, 1, 1], 8)
    out["mac_report"] = np.array([mr["original"], mr["dense_folded"], mr["grouped_folded"], mr["zero_padded"]],
                                 np.int64)
    mr3 = ref.mac_report([1, 16, 16, 3], [3, 1, 3, 4], 8)
    out["mac_report_rgb"] = np.array([mr3["original"], mr3["dense_folded"], mr3["grouped_folded"],
                                      mr3["zero_padded"]], np.int64)
    out["count_macs"] = np.array([ref.count_macs([1, 32, 64, 1], [5, 1, 1, 1]),
                                  ref.count_macs([2, 9, 11, 3], [3, 2, 3, 5], 2, 3)], np.int64)
    np.savez_compressed(os.path.join(HERE, "kats.npz"), **out)


def make_conv_cases():
    rng = np.random.default_rng(1002)
    out = {}
    cases = [(1, 6, 5, 2, 3, 2, 4, 1, 1), (2, 9, 11, 3, 3, 3, 5, 2, 2), (1, 12, 16, 3, 7, 7, 8, 2, 2),
             (2, 10, 10, 1, 3, 1, 2, 1, 1), (1, 15, 13, 4, 5, 3, 3, 3, 2), (1, 8, 8, 8, 1, 1, 16, 1, 1)]
    for i, (B, H, W, C, KH, KW, Co, sh, sw) in enumerate(cases):
        for kind in ("int", "float"):
            if kind == "int":
                x = rng.integers(-4, 5, size=(B, H, W, C)).astype(np.float32)
                w = rng.integers(-4, 5, size=(KH, KW, C, Co)).astype(np.float32)
                b = rng.integers(-4, 5, size=(Co,)).astype(np.float32)
            else:
                x = rng.uniform(-1, 1, size=(B, H, W, C)).astype(np.float32)
                w = rng.uniform(-1, 1, size=(KH, KW, C, Co)).astype(np.float32)
                b = rng.uniform(-1, 1, size=(Co,)).astype(np.float32)
            y = ref.conv2d(x, w, sh, sw)
            yb = ref.bias_add(y, b)
            tag = f"c{i}_{kind}"
            out[tag + "_x"], out[tag + "_w"], out[tag + "_b"] = x, w, b
            out[tag + "_y"], out[tag + "_yb"] = y, yb
            out[tag + "_stride"] = np.array([sh, sw], np.int64)
    np.savez_compressed(os.path.join(HERE, "conv_cases.npz"), **out)


def make_appendix_a():
    rng = np.random.default_rng(1001)
    out = {}
    for kind in ("float", "int"):
        if kind == "float":
            x = rng.uniform(-1, 1, (1, 32, 64, 1)).astype(np.float32)
            w = rng.uniform(-1, 1, (5, 1, 1, 1)).astype(np.float32)
            b = rng.uniform(-1, 1, (1,)).astype(np.float32)
        else:
            x = rng.integers(-4, 5, (1, 32, 64, 1)).astype(np.float32)
            w = rng.integers(-4, 5, (5, 1, 1, 1)).astype(np.float32)
            b = rng.integers(-4, 5, (1,)).astype(np.float32)
        plan, x_f, w_f, b_f = ref.apply_width_fold(x, w, b, 8)
        assert plan["status"] == "apply"
        y_folded = ref.reconstruct_output(ref.bias_add(ref.conv2d(x_f, w_f), b_f), 8)
        y_ref = ref.bias_add(ref.conv2d(x, w), b)
        for k, v in dict(x=x, w=w, b=b, x_f=x_f, w_f=w_f, b_f=b_f, y_folded=y_folded, y_ref=y_ref).items():
            out[f"{kind}_{k}"] = v
    np.savez_compressed(os.path.join(HERE, "appendix_a.npz"), **out)


def make_configs():
    out = {}
    for name, (B, H, W, C, KH, KW, Co, s, p, relu, dt) in CONFIGS.items():
        b_, h_, w_ = SMALL[name]
        rng = np.random.default_rng(1001 + list(CONFIGS).index(name))
        x = quantize(rng.uniform(-1, 1, (b_, h_, w_, C)).astype(np.float32), dt)
        w = quantize((rng.uniform(-1, 1, (KH, KW, C, Co)) / np.sqrt(KH * KW * C)).astype(np.float32), dt)
        b = quantize(rng.uniform(-1, 1, (Co,)).astype(np.float32), dt)
        out[f"{name}_x"], out[f"{name}_w"], out[f"{name}_b"] = x, w, b
        out[f"{name}_y"] = ref_conv(x, w, b, s, p, relu)
        xi = rng.integers(-4, 5, (b_, h_, w_, C)).astype(np.float32)
        wi = rng.integers(-4, 5, (KH, KW, C, Co)).astype(np.float32)
        bi = rng.integers(-4, 5, (Co,)).astype(np.float32)
        out[f"{name}_xi"], out[f"{name}_wi"], out[f"{name}_bi"] = xi, wi, bi
        out[f"{name}_yi"] = ref_conv(xi, wi, bi, s, p, relu)
        out[f"{name}_geom"] = np.array([KH, KW, C, Co, s, p, int(relu)], np.int64)
        out[f"{name}_dtype"] = np.array(dt)
    np.savez_compressed(os.path.join(HERE, "configs.npz"), **out)


if __name__ == "__main__":
    make_kats()
    make_conv_cases()
    make_appendix_a()
    make_configs()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)), "bytes")
