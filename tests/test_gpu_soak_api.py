"""Time-boxed randomised soak of the reference-facing operators on the device against the pinned oracle.

Each iteration draws one operator call with random shapes and real-valued data and checks it BIT FOR BIT:
  - conv2d(precision="exact") (padding, bias, ReLU, rectangular strides)  == oracle conv + bias_add + relu;
  - grouped_conv on a verified block-diagonal filter                        == oracle grouped_conv;
  - fold_tall_skinny(precision=None)                                        == gemm_ref (the reference's k-inner order);
  - fold_tall_skinny / gemm_as_conv1x1 on the tensor cores, integer data    == exact float64 matmul.
The budget is SOAK_API_SECONDS (default 20 s, so the suite stays short; `SOAK_API_SECONDS=600` for a long run).
"""
import os
import random
import time

import numpy as np
import pytest
import torch

import paper_2601_11608_b200 as wf

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32)).view(np.uint32)


def _exact_conv(rng, oracle):
    n, h, w, c = rng.randint(1, 3), rng.randint(1, 40), rng.randint(1, 48), rng.randint(1, 8)
    kh, kw, co = rng.randint(1, 11), rng.randint(1, 11), rng.randint(1, 40)
    sh, sw, ph, pw = rng.randint(1, 4), rng.randint(1, 4), rng.randint(0, 5), rng.randint(0, 5)
    if h + 2 * ph < kh or w + 2 * pw < kw:
        return None
    nr = np.random.default_rng(rng.randrange(1 << 30))
    x = nr.standard_normal((n, h, w, c)).astype(np.float32)
    wt = nr.standard_normal((kh, kw, c, co)).astype(np.float32)
    b = nr.standard_normal((co,)).astype(np.float32) if rng.random() < 0.6 else None
    relu = rng.random() < 0.4
    y = wf.conv2d(torch.from_numpy(x).cuda(), torch.from_numpy(wt).cuda(), sh, sw, padding=(ph, pw),
                  bias=None if b is None else torch.from_numpy(b).cuda(), relu=relu, precision="exact")
    ref = oracle.conv2d(oracle.pad(x, ph, pw), wt, sh, sw)
    if b is not None:
        ref = oracle.bias_add(ref, b)
    if relu:
        ref = oracle.relu(ref)
    np.testing.assert_array_equal(_bits(y.cpu().numpy()), _bits(ref), err_msg=f"conv2d exact {x.shape} {wt.shape}")
    return "conv2d_exact"


def _grouped(rng, oracle):
    F = rng.choice([1, 2, 3, 4, 8])
    n, h, c = rng.randint(1, 3), rng.randint(1, 24), rng.randint(1, 4)
    wf_, kh, co = rng.randint(1, 12), rng.randint(1, 5), rng.randint(1, 12)
    sh = rng.randint(1, 3)
    if h < kh:
        return None
    nr = np.random.default_rng(rng.randrange(1 << 30))
    w = nr.standard_normal((kh, 1, c, co)).astype(np.float32)
    wd = oracle.expand_filter_general(w, F)              # block-diagonal (KH, 1, F*C, F*Co)
    x = nr.standard_normal((n, h, wf_, F * c)).astype(np.float32)
    y = wf.grouped_conv(torch.from_numpy(x).cuda(), torch.from_numpy(wd).cuda(), F, sh, 1)
    ref = oracle.grouped_conv(x, wd, F, sh, 1)
    np.testing.assert_array_equal(_bits(y.cpu().numpy()), _bits(ref), err_msg=f"grouped {x.shape} F={F}")
    return "grouped_conv"


def _gemm_exact(rng, oracle):
    F = rng.choice([1, 2, 4, 8])
    M, K, N = F * rng.randint(1, 300), rng.randint(1, 24), rng.randint(1, 48)
    nr = np.random.default_rng(rng.randrange(1 << 30))
    a = torch.from_numpy(nr.standard_normal((M, K)).astype(np.float32)).cuda()
    b = torch.from_numpy(nr.standard_normal((K, N)).astype(np.float32)).cuda()
    c = wf.fold_tall_skinny(a, b, F)
    ref = wf.gemm_ref(a, b)
    assert torch.equal(c, ref), f"fold_tall_skinny exact M={M} K={K} N={N} F={F}"
    return "gemm_exact"


def _gemm_tensor(rng, oracle):
    F = rng.choice([1, 2, 4, 8])
    K, N = rng.choice([1, 2, 3, 4, 6, 8]), rng.choice([32, 64, 96, 128, 160, 256])
    M = F * rng.randint(1, 5000)
    prec = rng.choice(["bf16", "f16"])
    g = torch.Generator(device="cuda").manual_seed(rng.randrange(1 << 30))
    a = torch.randint(-4, 5, (M, K), generator=g, device="cuda").float()
    b = torch.randint(-4, 5, (K, N), generator=g, device="cuda").float()
    ref = a.double() @ b.double()
    try:
        if rng.random() < 0.5:
            c, op = wf.fold_tall_skinny(a, b, F, precision=prec, out_dtype=torch.float32), "fold_tall_skinny"
        else:
            c, op = wf.gemm_as_conv1x1(a, b, precision=prec, out_dtype=torch.float32), "gemm_as_conv1x1"
    except wf.UnsupportedError:
        return None
    assert torch.equal(c.double(), ref), f"{op} {prec} M={M} K={K} N={N} F={F}"
    return op


def test_api_soak(oracle):
    budget = float(os.environ.get("SOAK_API_SECONDS", "20"))
    rng = random.Random(int(os.environ.get("SOAK_API_SEED", "1608")))
    ops = [_exact_conv, _grouped, _gemm_exact, _gemm_tensor]
    done = {}
    t_end = time.time() + budget
    while time.time() < t_end:
        name = rng.choice(ops)(rng, oracle)
        if name:
            done[name] = done.get(name, 0) + 1
    print("api soak:", done)
    assert all(done.get(k, 0) > 0 for k in ("conv2d_exact", "grouped_conv", "gemm_exact")), done
