"""Randomised geometries through the folded tcgen05 kernel (and the unfolded variant).

Seeded random convolutions -- batch 1-4, H 8-72, W 8-96, Cin 1-4, square
kernels 1-11, stride 1-4, padding 0-K/2, Cout 32-128, bf16 / fp16 / TF32,
optional ReLU -- planned by the generalized fold (every planner path: fold
factor, group size, K-step schedule, N-tiling, producer, stage tiles) and
compared EXACTLY with a float64 conv: integer-valued inputs, weights and bias
keep every product and partial sum exact in the fp32 accumulator, so any
indexing, layout, masking or synchronisation error shows up as a mismatch.
Geometries the fold does not apply to (the planner's fallback reasons) are
counted, not run.
"""
import random
import zlib

import pytest
import torch

import paper_2601_11608_b200 as wf

pytestmark = pytest.mark.gpu

TDT = {"bf16": torch.bfloat16, "f16": torch.float16, "tf32": torch.float32}


def _cases(count=160, seed=2601):
    rng = random.Random(seed)
    out = []
    while len(out) < count:
        n, h, w = rng.randint(1, 4), rng.randint(8, 72), rng.randint(8, 96)
        c, k, s = rng.choice([1, 2, 3, 4]), rng.choice([1, 2, 3, 5, 7, 11]), rng.randint(1, 4)
        p = rng.randint(0, k // 2)
        co, dt, relu = rng.choice([32, 64, 96, 128]), rng.choice(["bf16", "f16", "tf32"]), rng.random() < 0.3
        if (h + 2 * p - k) // s + 1 < 1 or (w + 2 * p - k) // s + 1 < 1:
            continue
        variant = "unfolded" if (dt != "tf32" and rng.random() < 0.25) else "fold"
        out.append((n, h, w, c, k, s, p, co, dt, relu, variant))
    return out


CASES = _cases()


def _f64(x, w, b, s, p, relu):
    # cuDNN off: its float64 algorithms for some shapes (e.g. 8 channels, large batches) are not exact on
    # integer data (-17.999999999999996 for -18, found by tools/fuzz_soak.py); the native im2col + DGEMM is
    with torch.backends.cudnn.flags(enabled=False):
        return _f64_native(x, w, b, s, p, relu)


def _f64_native(x, w, b, s, p, relu):
    y = torch.nn.functional.conv2d(x.double().permute(0, 3, 1, 2), w.double().permute(3, 2, 0, 1), b.double(),
                                   stride=s, padding=p).permute(0, 2, 3, 1)
    return torch.relu(y) if relu else y


@pytest.mark.parametrize("case", CASES, ids=[f"n{c[0]}_{c[1]}x{c[2]}x{c[3]}_k{c[4]}s{c[5]}p{c[6]}_co{c[7]}_{c[8]}"
                                             f"{'_relu' if c[9] else ''}_{c[10]}" for c in CASES])
def test_random_geometry_exact(case):
    n, h, w, c, k, s, p, co, dt, relu, variant = case
    g = torch.Generator(device="cuda").manual_seed(zlib.crc32(repr(case).encode()))
    tdt = TDT[dt]
    x = torch.randint(-3, 4, (n, h, w, c), generator=g, device="cuda").to(tdt)
    wt = torch.randint(-3, 4, (k, k, c, co), generator=g, device="cuda").to(tdt)
    b = torch.randint(-8, 9, (co,), generator=g, device="cuda").float()
    try:
        conv = wf.FoldedConv2d(wt, b, x.shape, stride=s, padding=p, dtype=tdt, variant=variant)
    except wf.UnsupportedError as e:  # the planner's fallback (FactorTooLarge, NotProfitable, ...)
        pytest.skip(f"fold not applicable: {e}")
    y = conv(x, relu=relu, out_dtype=torch.float32)
    ref = _f64(x, wt, b, s, p, relu)
    assert y.shape == ref.shape
    bad = (y.double() != ref)
    assert not bad.any(), (f"{int(bad.sum())} of {bad.numel()} outputs differ; plan "
                           f"{ {key: conv.device_plan[key] for key in ('f', 'r', 'group_size', 'n_tiles', 'producer', 'kstep_mode', 'stage_tiles', 'wbox')} }")


def test_fuzz_covers_the_planner():
    """The random set exercises every dtype, both variants and most fold applications."""
    dts = {c[8] for c in CASES}
    assert dts == {"bf16", "f16", "tf32"}
    assert {c[10] for c in CASES} == {"fold", "unfolded"}
    applied = 0
    from paper_2601_11608_b200 import _core
    for n, h, w, c, k, s, p, co, dt, relu, variant in CASES:
        try:
            _core.FoldedConv([n, h, w, c], [k, k, c, co], s, s, p, p, dt, 0, 0, variant)
            applied += 1
        except wf.UnsupportedError:
            pass
    assert applied >= 0.85 * len(CASES)


# ---- second set: rectangular kernels, unequal strides / padding, wider rows, and the planner knobs
KNOBS = [{}, {"WF_KPAIR": "0"}, {"WF_KPAIR": "1"}, {"WF_TPS": "1"}, {"WF_TPS": "2"}, {"WF_MCAST": "1"},
         {"WF_MCAST": "0"}, {"WF_GATHER": "1"}, {"WF_GATHER": "2"}, {"WF_RING": "1"}, {"WF_PLANES": "0"},
         {"WF_NACC": "2"}, {"WF_EPI_PP": "1"}, {"WF_PDL": "0"}]


def _cases2(count=120, seed=11608):
    rng = random.Random(seed)
    out = []
    while len(out) < count:
        n, h, w = rng.randint(1, 6), rng.randint(6, 64), rng.randint(6, 240)
        c = rng.choice([1, 2, 3, 4, 6, 8])
        kh, kw = rng.choice([1, 2, 3, 5, 7]), rng.choice([1, 2, 3, 5, 7, 11])
        sh, sw = rng.randint(1, 3), rng.randint(1, 4)
        ph, pw = rng.randint(0, kh // 2), rng.randint(0, kw // 2)
        co, dt, relu = rng.choice([32, 64, 96, 128, 160, 256]), rng.choice(["bf16", "f16", "tf32"]), rng.random() < 0.3
        if (h + 2 * ph - kh) // sh + 1 < 1 or (w + 2 * pw - kw) // sw + 1 < 1:
            continue
        out.append((n, h, w, c, kh, kw, sh, sw, ph, pw, co, dt, relu, rng.randrange(len(KNOBS))))
    return out


CASES2 = _cases2()


@pytest.mark.parametrize("case", CASES2, ids=[f"n{c[0]}_{c[1]}x{c[2]}x{c[3]}_k{c[4]}x{c[5]}_s{c[6]}x{c[7]}_p{c[8]}x{c[9]}"
                                               f"_co{c[10]}_{c[11]}{'_relu' if c[12] else ''}_knob{c[13]}"
                                               for c in CASES2])
def test_random_geometry_and_knobs_exact(case, monkeypatch):
    n, h, w, c, kh, kw, sh, sw, ph, pw, co, dt, relu, knob = case
    for key, val in KNOBS[knob].items():
        monkeypatch.setenv(key, val)
    g = torch.Generator(device="cuda").manual_seed(zlib.crc32(repr(case).encode()))
    tdt = TDT[dt]
    x = torch.randint(-3, 4, (n, h, w, c), generator=g, device="cuda").to(tdt)
    wt = torch.randint(-3, 4, (kh, kw, c, co), generator=g, device="cuda").to(tdt)
    b = torch.randint(-8, 9, (co,), generator=g, device="cuda").float()
    try:
        conv = wf.FoldedConv2d(wt, b, x.shape, stride=(sh, sw), padding=(ph, pw), dtype=tdt)
    except wf.UnsupportedError as e:
        pytest.skip(f"fold not applicable: {e}")
    y = conv(x, relu=relu, out_dtype=torch.float32)
    with torch.backends.cudnn.flags(enabled=False):  # exact float64 reference (see _f64)
        ref = torch.nn.functional.conv2d(x.double().permute(0, 3, 1, 2), wt.double().permute(3, 2, 0, 1),
                                         b.double(), stride=(sh, sw), padding=(ph, pw)).permute(0, 2, 3, 1)
    if relu:
        ref = torch.relu(ref)
    bad = (y.double() != ref)
    assert not bad.any(), (f"{int(bad.sum())} of {bad.numel()} outputs differ with {KNOBS[knob]}; plan "
                           f"{ {key: conv.device_plan[key] for key in ('f', 'r', 'group_size', 'n_tiles', 'producer', 'kstep_mode', 'stage_tiles', 'wbox')} }")


TOL = {"bf16": 1e-2, "f16": 1e-2, "tf32": 1e-3}


@pytest.mark.parametrize("case", CASES[:48], ids=[f"real_n{c[0]}_{c[1]}x{c[2]}x{c[3]}_k{c[4]}s{c[5]}p{c[6]}_co{c[7]}_{c[8]}"
                                                  f"_{c[10]}" for c in CASES[:48]])
def test_random_geometry_real_data_within_tolerance(case):
    """Real-valued data: normwise max|y - ref| / max|ref| within the north-star tolerance (bf16/fp16 1e-2,
    TF32 1e-3) of a float64 conv of the same (device-representable) inputs."""
    n, h, w, c, k, s, p, co, dt, relu, variant = case
    g = torch.Generator(device="cuda").manual_seed(zlib.crc32(repr(case).encode()) ^ 0x5A5A)
    tdt = TDT[dt]
    x = (torch.rand((n, h, w, c), generator=g, device="cuda") * 2 - 1).to(tdt)
    wt = ((torch.rand((k, k, c, co), generator=g, device="cuda") * 2 - 1) / (k * k * c) ** 0.5).to(tdt)
    b = torch.rand((co,), generator=g, device="cuda") * 2 - 1
    try:
        conv = wf.FoldedConv2d(wt, b, x.shape, stride=s, padding=p, dtype=tdt, variant=variant)
    except wf.UnsupportedError as e:
        pytest.skip(f"fold not applicable: {e}")
    # every output type the epilogue writes (bf16 / fp16 rounding counts against the tolerance)
    odt = (torch.float32, torch.bfloat16, torch.float16)[zlib.crc32(repr(case).encode()) % 3]
    y = conv(x, relu=relu, out_dtype=odt).double()
    ref = _f64(x, wt, b, s, p, relu)
    err = ((y - ref).abs().max() / ref.abs().max().clamp_min(1e-30)).item()
    tol = TOL[dt] if odt == torch.float32 else 1e-2
    assert err <= tol, f"normwise rel err {err:.3e} > {tol} (out {odt})"


@pytest.mark.parametrize("case", CASES2[:64], ids=[f"real_n{c[0]}_{c[1]}x{c[2]}x{c[3]}_k{c[4]}x{c[5]}_s{c[6]}x{c[7]}"
                                                   f"_p{c[8]}x{c[9]}_co{c[10]}_{c[11]}_knob{c[13]}" for c in CASES2[:64]])
def test_random_geometry_and_knobs_real_data(case, monkeypatch):
    """Real-valued data through the knob set: within tolerance and free of NaN (a schedule that read
    unloaded shared memory would multiply garbage by zero filter taps and could produce NaN)."""
    n, h, w, c, kh, kw, sh, sw, ph, pw, co, dt, relu, knob = case
    for key, val in KNOBS[knob].items():
        monkeypatch.setenv(key, val)
    g = torch.Generator(device="cuda").manual_seed(zlib.crc32(repr(case).encode()) ^ 0xA5A5)
    tdt = TDT[dt]
    x = (torch.rand((n, h, w, c), generator=g, device="cuda") * 2 - 1).to(tdt)
    wt = ((torch.rand((kh, kw, c, co), generator=g, device="cuda") * 2 - 1) / (kh * kw * c) ** 0.5).to(tdt)
    b = torch.rand((co,), generator=g, device="cuda") * 2 - 1
    try:
        conv = wf.FoldedConv2d(wt, b, x.shape, stride=(sh, sw), padding=(ph, pw), dtype=tdt)
    except wf.UnsupportedError as e:
        pytest.skip(f"fold not applicable: {e}")
    y = conv(x, relu=relu, out_dtype=torch.float32).double()
    with torch.backends.cudnn.flags(enabled=False):  # exact float64 reference (see _f64)
        ref = torch.nn.functional.conv2d(x.double().permute(0, 3, 1, 2), wt.double().permute(3, 2, 0, 1),
                                         b.double(), stride=(sh, sw), padding=(ph, pw)).permute(0, 2, 3, 1)
    if relu:
        ref = torch.relu(ref)
    assert torch.isfinite(y).all()
    err = ((y - ref).abs().max() / ref.abs().max().clamp_min(1e-30)).item()
    assert err <= TOL[dt], f"normwise rel err {err:.3e} > {TOL[dt]} with {KNOBS[knob]}"


def _cases3(count=40, seed=31337):
    """Larger batches of small images: many tiles per CTA (A-stage ring, accumulator buffers and barrier
    phases wrap many times) for unusual plans."""
    rng = random.Random(seed)
    out = []
    while len(out) < count:
        n, h, w = rng.randint(64, 320), rng.randint(6, 40), rng.randint(6, 64)
        c, k, s = rng.choice([1, 2, 3, 4]), rng.choice([1, 3, 5, 7]), rng.randint(1, 3)
        p = rng.randint(0, k // 2)
        co, dt = rng.choice([32, 64, 96, 128, 192]), rng.choice(["bf16", "f16", "tf32"])
        if (h + 2 * p - k) // s + 1 < 1 or (w + 2 * p - k) // s + 1 < 1:
            continue
        out.append((n, h, w, c, k, s, p, co, dt, rng.random() < 0.3, rng.randrange(len(KNOBS))))
    return out


CASES3 = _cases3()


@pytest.mark.parametrize("case", CASES3, ids=[f"n{c[0]}_{c[1]}x{c[2]}x{c[3]}_k{c[4]}s{c[5]}p{c[6]}_co{c[7]}_{c[8]}"
                                               f"_knob{c[10]}" for c in CASES3])
def test_random_steady_state_exact(case, monkeypatch):
    n, h, w, c, k, s, p, co, dt, relu, knob = case
    for key, val in KNOBS[knob].items():
        monkeypatch.setenv(key, val)
    g = torch.Generator(device="cuda").manual_seed(zlib.crc32(repr(case).encode()))
    tdt = TDT[dt]
    x = torch.randint(-3, 4, (n, h, w, c), generator=g, device="cuda").to(tdt)
    wt = torch.randint(-3, 4, (k, k, c, co), generator=g, device="cuda").to(tdt)
    b = torch.randint(-8, 9, (co,), generator=g, device="cuda").float()
    try:
        conv = wf.FoldedConv2d(wt, b, x.shape, stride=s, padding=p, dtype=tdt)
    except wf.UnsupportedError as e:
        pytest.skip(f"fold not applicable: {e}")
    y = conv(x, relu=relu, out_dtype=torch.float32)
    ref = _f64(x, wt, b, s, p, relu)
    bad = (y.double() != ref).reshape(n, -1).any(dim=1)
    assert not bad.any(), (f"images {bad.nonzero().flatten().tolist()[:8]} differ with {KNOBS[knob]}; plan "
                           f"{ {key: conv.device_plan[key] for key in ('f', 'r', 'n_tiles', 'producer', 'kstep_mode', 'stage_tiles', 'wbox')} }")
