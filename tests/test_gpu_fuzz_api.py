"""Randomised checks of the reference-facing operators on the device, against the pinned oracle.

- `conv2d(..., precision="exact")` (the reference's fp32 order kh -> kw -> ci, no FMA, on CUDA cores)
  equals the oracle's restatement of `widthfold::conv2d` BIT FOR BIT on random real-valued data, with
  and without padding / bias / ReLU;
- the fold index transforms (`fold_input_general`, `unfold_input_general`, `expand_filter_general`)
  equal the oracle bit for bit (compared as uint32 patterns);
- `fold_tall_skinny` on the tensor cores is exact on integer data for random (M, K, N, F).
"""
import random
import zlib

import numpy as np
import pytest
import torch

import paper_2601_11608_b200 as wf

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32)).view(np.uint32)


def _conv_cases(count=40, seed=7):
    rng = random.Random(seed)
    out = []
    while len(out) < count:
        n, h, w, c = rng.randint(1, 3), rng.randint(3, 20), rng.randint(3, 24), rng.randint(1, 5)
        kh, kw, co = rng.randint(1, 5), rng.randint(1, 5), rng.randint(1, 9)
        sh, sw = rng.randint(1, 3), rng.randint(1, 3)
        ph, pw = rng.randint(0, 2), rng.randint(0, 2)
        if (h + 2 * ph - kh) // sh + 1 < 1 or (w + 2 * pw - kw) // sw + 1 < 1:
            continue
        out.append((n, h, w, c, kh, kw, co, sh, sw, ph, pw, rng.random() < 0.5, rng.random() < 0.3))
    return out


@pytest.mark.parametrize("case", _conv_cases())
def test_exact_conv_bitwise_vs_oracle(oracle, case):
    n, h, w, c, kh, kw, co, sh, sw, ph, pw, use_bias, relu = case
    rng = np.random.default_rng(zlib.crc32(repr(case).encode()))
    x = rng.standard_normal((n, h, w, c)).astype(np.float32)
    wt = rng.standard_normal((kh, kw, c, co)).astype(np.float32)
    b = rng.standard_normal((co,)).astype(np.float32) if use_bias else None
    y = wf.conv2d(torch.from_numpy(x).cuda(), torch.from_numpy(wt).cuda(), sh, sw, padding=(ph, pw),
                  bias=None if b is None else torch.from_numpy(b).cuda(), relu=relu, precision="exact")
    ref = oracle.conv2d(oracle.pad(x, ph, pw), wt, sh, sw)
    if b is not None:
        ref = oracle.bias_add(ref, b)
    if relu:
        ref = oracle.relu(ref)
    np.testing.assert_array_equal(_bits(y.cpu().numpy()), _bits(ref))


@pytest.mark.parametrize("seed", range(12))
def test_fold_transforms_bitwise_vs_oracle(oracle, seed):
    rng = random.Random(seed)
    F = rng.choice([1, 2, 3, 4, 8])
    n, h, c = rng.randint(1, 3), rng.randint(1, 9), rng.randint(1, 5)
    w = F * rng.randint(1, 7)
    nrng = np.random.default_rng(seed)
    x = nrng.standard_normal((n, h, w, c)).astype(np.float32)
    xf = wf.fold_input_general(torch.from_numpy(x).cuda(), F)
    np.testing.assert_array_equal(_bits(xf.cpu().numpy()), _bits(oracle.fold_input_general(x, F)))
    back = wf.unfold_input_general(xf, F)
    np.testing.assert_array_equal(_bits(back.cpu().numpy()), _bits(x))
    kh, co = rng.randint(1, 4), rng.randint(1, 6)
    wt = nrng.standard_normal((kh, 1, c, co)).astype(np.float32)
    we = wf.expand_filter_general(torch.from_numpy(wt).cuda(), F)
    np.testing.assert_array_equal(_bits(we.cpu().numpy()), _bits(oracle.expand_filter_general(wt, F)))


@pytest.mark.parametrize("seed", range(16))
def test_tall_skinny_gemm_exact_on_integers(seed):
    rng = random.Random(seed)
    F = rng.choice([1, 2, 4, 8])
    K = rng.choice([1, 2, 3, 4, 6, 8])
    N = rng.choice([32, 64, 96, 128])
    M = F * rng.randint(1, 4000)
    prec = rng.choice(["bf16", "f16"])
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.randint(-4, 5, (M, K), generator=g, device="cuda").float()
    b = torch.randint(-4, 5, (K, N), generator=g, device="cuda").float()
    try:
        c = wf.fold_tall_skinny(a, b, F, precision=prec, out_dtype=torch.float32)
    except wf.UnsupportedError as e:
        pytest.skip(f"fold not applicable: {e}")
    ref = a.double() @ b.double()
    assert torch.equal(c.double(), ref)
