"""GPU parity: the sm_100a kernels vs the pinned oracle / reference goldens.

Tolerances (north star): integer-valued data exact; bf16/fp16 normwise
max|y - y_ref| / max|y_ref| <= 1e-2; TF32 <= 1e-3; the exact-fp32 CUDA-core
path and all index transforms bit-exact. Inputs are device-representable
(quantised) values, so differences isolate accumulation order and output
rounding.
"""
import numpy as np
import pytest
import torch

import paper_2601_11608_b200 as wf
from paper_2601_11608_b200 import _abi as A
from tests.test_oracle import CONFIG_GEOM

pytestmark = pytest.mark.gpu

TOL = {"bf16": 1e-2, "f16": 1e-2, "f32": 1e-3}
TDT = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32}


def normrel(y, ref):
    y = np.asarray(y, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.max(np.abs(y - ref)) / max(np.max(np.abs(ref)), 1e-30))


def chunk_perm(col, ch):
    """Accumulator column -> output column inside an epilogue chunk (plan.hpp chunk_perm)."""
    c, w = divmod(col, ch)
    return c * ch + (ch // 4) * ((w % 8) // 2) + 2 * (w // 8) + (w % 2)


def cuda(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda").to(dtype)


def test_exact_conv_matches_reference_bitwise(golden_conv):
    tags = sorted({k.rsplit("_", 1)[0] for k in golden_conv if k.endswith("_x")})
    for tag in tags:
        g = {k[len(tag) + 1:]: v for k, v in golden_conv.items() if k.startswith(tag + "_")}
        sh, sw = (int(v) for v in g["stride"])
        y = wf.conv2d(g["x"], g["w"], sh, sw)  # numpy in -> reference semantics (exact fp32)
        assert isinstance(y, np.ndarray)
        np.testing.assert_array_equal(y.view(np.uint32), g["y"].view(np.uint32), err_msg=tag)
        yb = wf.bias_add(y, g["b"])
        np.testing.assert_array_equal(yb.view(np.uint32), g["yb"].view(np.uint32), err_msg=tag)
        yb2 = wf.conv2d(g["x"], g["w"], sh, sw, bias=g["b"])
        np.testing.assert_array_equal(yb2.view(np.uint32), g["yb"].view(np.uint32), err_msg=tag)


def test_appendix_a_on_device(golden_appendix):
    for kind in ("float", "int"):
        g = {k[len(kind) + 1:]: v for k, v in golden_appendix.items() if k.startswith(kind + "_")}
        plan, x_f, w_f, b_f = wf.apply_width_fold(g["x"], g["w"], g["b"], 8)
        assert plan["status"] == "apply" and plan["folded_input_shape"] == [1, 32, 8, 8]
        np.testing.assert_array_equal(x_f, g["x_f"])
        np.testing.assert_array_equal(w_f, g["w_f"])
        np.testing.assert_array_equal(b_f, g["b_f"])
        y = wf.reconstruct_output(wf.bias_add(wf.conv2d(x_f, w_f), b_f), 8)
        np.testing.assert_array_equal(y, g["y_folded"])


def test_fallback_keeps_inputs():
    x = np.zeros((1, 4, 7, 1), np.float32)
    plan, x2, w2, b2 = wf.apply_width_fold(x, np.zeros((3, 1, 1, 1), np.float32), np.zeros(1, np.float32), 8)
    assert plan["status"] == "fallback" and plan["reason"] == "WidthNotDivisible"
    np.testing.assert_array_equal(x2, x)
    with pytest.raises(ValueError):
        wf.fold_input(np.zeros((1, 2, 7, 1), np.float32), 2)


def test_fold_views_are_zero_copy():
    x = torch.randn(2, 8, 32, 3, device="cuda")
    xf = wf.fold_input_general(x, 16)
    assert xf.data_ptr() == x.data_ptr() and tuple(xf.shape) == (2, 8, 2, 48)
    back = wf.unfold_input_general(xf, 16)
    assert back.data_ptr() == x.data_ptr() and torch.equal(back, x)
    y = torch.randn(2, 5, 14, 512, device="cuda")
    r = wf.reconstruct_output(y, 8)
    assert r.data_ptr() == y.data_ptr() and tuple(r.shape) == (2, 5, 112, 64)


def test_expand_filters_bitwise(golden_kats, golden_configs, oracle):
    np.testing.assert_array_equal(wf.expand_filter_general(golden_kats["expand_general_in"], 4),
                                  golden_kats["expand_general_out_f4"])
    np.testing.assert_array_equal(wf.expand_filter(golden_kats["expand_in"], 2), golden_kats["expand_out"])
    np.testing.assert_array_equal(wf.replicate_bias(np.array([1, 2], np.float32), 3), golden_kats["replicate"])
    for name, f in CONFIG_GEOM.items():
        KH, KW, C, Co, s, p, relu = (int(v) for v in golden_configs[f"{name}_geom"])
        w = golden_configs[f"{name}_w"]
        np.testing.assert_array_equal(wf.expand_filter_folded(w, f, s, p), oracle.expand_filter_folded(w, f, s, p),
                                      err_msg=name)
    with pytest.raises(wf.IllegalFoldError):
        wf.expand_filter_general(np.zeros((3, 3, 1, 1), np.float32), 2)


def _config_run(golden_configs, name, suffix, out_dtype=None, variant="fold", flags=0):
    KH, KW, C, Co, s, p, relu = (int(v) for v in golden_configs[f"{name}_geom"])
    dt = str(golden_configs[f"{name}_dtype"])
    x, w, b = (golden_configs[f"{name}_{k}{suffix}"] for k in ("x", "w", "b"))
    tdt = TDT[dt]
    conv = wf.FoldedConv2d(cuda(w, tdt), cuda(b), x.shape, stride=s, padding=p, dtype=tdt, variant=variant)
    y = conv._forward(cuda(x, tdt), relu=bool(relu), out_dtype=out_dtype, flags=flags)
    torch.cuda.synchronize()
    return y.float().cpu().numpy(), golden_configs[f"{name}_y{suffix}"], dt, conv


@pytest.mark.parametrize("name", list(CONFIG_GEOM))
def test_tensor_core_conv_configs_within_tolerance(golden_configs, name):
    y, ref, dt, conv = _config_run(golden_configs, name, "")
    assert y.shape == ref.shape
    err = normrel(y, ref)
    assert err <= TOL[dt], f"{name}: normwise rel {err:.3e} > {TOL[dt]} (plan {conv.device_plan})"


VARIANT_ENVS = [
    {"WF_KPAIR": "0"}, {"WF_KPAIR": "1"},          # 32-byte covers / cross-kh core-column pairs
    {"WF_CTA_PAIR": "1"},                           # cta_group::2 pairs (opt-in)
    {"WF_TPS": "1"}, {"WF_TPS": "2"}, {"WF_TPS": "4"},  # M tiles per A stage
    {"WF_NACC": "2"},                               # two accumulator buffers
    {"WF_EPI_PP": "1"}, {"WF_EPI_PP": "0"},         # epilogue warp groups alternate tiles / share each tile
]


@pytest.mark.parametrize("env", VARIANT_ENVS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
@pytest.mark.parametrize("name", list(CONFIG_GEOM))
def test_tensor_core_conv_integer_data_exact(golden_configs, name, env, monkeypatch):
    """Every schedule / pipeline variant of the kernel is exact on integer data."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    y, ref, dt, conv = _config_run(golden_configs, name, "i", out_dtype=torch.float32)
    np.testing.assert_array_equal(y, ref, err_msg=f"{name} plan {conv.device_plan}")


def _unpack_and_check(conv, w, s, p, oracle):
    """Rebuild W'(kh, kw', fi*C+c, j*Co+co) from the packed operand; every
    nonzero of the expansion must be stored exactly once.

    Packed header: per MMA a 16-byte entry (a_off, b_off, meta, tmem_col),
    meta = kh | u << 8 | slot << 16 | (N/8) << 22 | acc << 31, the
    accumulator-slot -> group order (int32), then per entry two words
    kh | c << 8 | mask << 16 naming the window-row core column c of filter row
    kh that the entry's core column 0 / 1 holds, for the slots in mask. B block
    of an entry: [core col 0..1][N rows][8 elements]; row n is accumulator
    column slot*Ng + n = group order[slot + n // Ng], output column
    chunk_perm(n % Ng).
    """
    KH, KW, C, Co = w.shape
    d = conv.device_plan
    f, gs, ch = d["f"], d["group_size"], d["epi_chunk"]
    Ng = gs * Co
    G = d["n_groups"]
    wexp = oracle.expand_filter_folded(w, f, s, p)  # (KH, KW', f*C, r*Co)
    kwf = wexp.shape[1]
    E2 = 8  # 2-byte elements per 16-byte core column
    raw = conv.packed.cpu().numpy()
    n_ent = d["mma_entries"]
    table = raw[: n_ent * 16].view(np.uint32).reshape(n_ent, 4)
    order = raw[n_ent * 16: n_ent * 16 + 4 * G].view(np.int32)
    ccw = raw[n_ent * 16 + 4 * G: n_ent * 24 + 4 * G].view(np.uint32).reshape(n_ent, 2)
    assert sorted(order.tolist()) == list(range(G))
    base = (n_ent * 24 + 4 * G + 127) // 128 * 128
    pair = d["cta_pair"]
    b_total = len(raw) - base
    recon = np.zeros((KH, kwf * f * C + 2 * E2, wexp.shape[3]), np.float64)
    # N-tile of every entry (first group, B base = the B bytes of the tiles before it)
    nts = np.array(A.schedule_describe(A.make_desc(*conv.input_shape, KH, KW, Co, s, s, p, p), 0, 0,
                                       A.WF_BF16)["ntiles"]).reshape(-1, 6)
    assert len(nts) == d["n_tiles"]
    tile_g0, tile_b0, bcur = np.zeros(n_ent, np.int64), np.zeros(n_ent, np.int64), 0
    for (_, _, e0, ne, g0, _) in nts:
        tile_g0[e0:e0 + ne] = g0
        tile_b0[e0:e0 + ne] = bcur
        bcur += int(sum(((table[i][2] >> 22) & 0x1FF) * 8 * 32 for i in range(e0, e0 + ne)))
    assert bcur == b_total
    for ei, ((a_off, b_off, meta, col), words) in enumerate(zip(table, ccw)):
        slot = tile_g0[ei] + ((meta >> 16) & 0x3F)
        N = ((meta >> 22) & 0x1FF) * 8
        b_off = b_off + tile_b0[ei]
        assert col == (slot - tile_g0[ei]) * Ng
        assert (words[0] & 0xFF, (words[0] >> 8) & 0xFF) == (meta & 0xFF, (meta >> 8) & 0xFF)
        if pair == 2:  # CTA r of the pair holds rows [r*N/2, (r+1)*N/2) of every block
            halves = []
            for r in range(2):
                o = base + r * (b_total // 2) + b_off // 2
                halves.append(raw[o: o + N * 16].view(np.uint16).reshape(2, N // 2, 8))
            blk = np.concatenate(halves, axis=1)
        else:
            blk = raw[base + b_off: base + b_off + N * 32].view(np.uint16).reshape(2, N, 8)
        vals = (blk.astype(np.uint32) << 16).view(np.float32)
        for cc in range(2):
            kh, c, mask = words[cc] & 0xFF, (words[cc] >> 8) & 0xFF, words[cc] >> 16
            for n in range(N):
                if not (mask >> (n // Ng)) & 1:
                    assert not vals[cc, n].any()
                    continue
                ocol = order[slot + n // Ng] * Ng + chunk_perm(n % Ng, ch)
                recon[kh, c * E2: c * E2 + E2, ocol] += vals[cc, n]
    assert not recon[:, kwf * f * C:].any()
    np.testing.assert_array_equal(recon[:, : kwf * f * C].reshape(wexp.shape[0], kwf, f * C, -1), wexp)


@pytest.mark.parametrize("kpair", ["0", "1"])
def test_packed_operand_unpacks_to_the_expansion(oracle, monkeypatch, kpair):
    """The once-packed tcgen05 B operand holds exactly W'(kh, kw', fi*C+c, j*Co+co),
    with the legacy 32-byte K-step cover and with cross-kh core-column pairs."""
    monkeypatch.setenv("WF_KPAIR", kpair)
    rng = np.random.default_rng(5)
    for (KH, KW, C, Co, s, p, hw) in [(7, 7, 3, 64, 2, 3, 64), (3, 3, 3, 64, 1, 1, 32), (11, 11, 3, 96, 4, 0, 67),
                                      (3, 3, 3, 32, 2, 1, 32)]:
        w = rng.integers(-8, 9, (KH, KW, C, Co)).astype(np.float32)
        conv = wf.FoldedConv2d(cuda(w, torch.bfloat16), None, (2, hw, hw, 3), stride=s, padding=p,
                               dtype=torch.bfloat16)
        _unpack_and_check(conv, w, s, p, oracle)


@pytest.mark.parametrize("batch,h,w", [(3, 36, 48), (1, 224, 224), (5, 20, 32), (2, 9, 16)])
def test_partial_tiles_and_odd_shapes(oracle, batch, h, w):
    """OH not a multiple of the 8-row M tile, tiny images, batch tails: exact on integers."""
    rng = np.random.default_rng(batch * 100 + h)
    x = rng.integers(-4, 5, (batch, h, w, 3)).astype(np.float32)
    wt = rng.integers(-4, 5, (7, 7, 3, 64)).astype(np.float32)
    b = rng.integers(-4, 5, (64,)).astype(np.float32)
    conv = wf.FoldedConv2d(cuda(wt, torch.bfloat16), cuda(b), x.shape, stride=2, padding=3, dtype=torch.bfloat16)
    y = conv(cuda(x, torch.bfloat16), out_dtype=torch.float32).cpu().numpy()
    ref = oracle.conv_padded(x, wt, b, 2, 3)
    np.testing.assert_array_equal(y, ref)


def test_epilogue_variants(oracle):
    rng = np.random.default_rng(9)
    x = rng.uniform(-1, 1, (2, 32, 32, 3)).astype(np.float32)
    w = (rng.uniform(-1, 1, (3, 3, 3, 32)) / 5).astype(np.float32)
    b = rng.uniform(-1, 1, (32,)).astype(np.float32)
    xq = cuda(x, torch.float16)
    wq = cuda(w, torch.float16)
    xs, ws = xq.float().cpu().numpy(), wq.float().cpu().numpy()
    conv = wf.FoldedConv2d(wq, cuda(b), x.shape, stride=2, padding=1, dtype=torch.float16)
    for relu in (False, True):
        for bias in (False, True):
            for od in (torch.float16, torch.float32, torch.bfloat16):
                y = conv(xq, relu=relu, bias=bias, out_dtype=od).float().cpu().numpy()
                ref = oracle.conv_padded(xs, ws, b if bias else None, 2, 1, relu)
                assert normrel(y, ref) <= 1e-2, (relu, bias, od)


def test_full_size_sampled_images(oracle):
    """Full 224x224 geometry, batch 6: compare two sampled images with the oracle."""
    rng = np.random.default_rng(1234)
    for (KH, Co, s, p, dt) in ((7, 64, 2, 3, torch.bfloat16), (3, 64, 1, 1, torch.bfloat16),
                               (3, 32, 2, 1, torch.float16)):
        x = torch.from_numpy(rng.uniform(-1, 1, (6, 224, 224, 3)).astype(np.float32)).cuda().to(dt)
        w = torch.from_numpy((rng.uniform(-1, 1, (KH, KH, 3, Co)) / KH / 2).astype(np.float32)).cuda().to(dt)
        b = torch.from_numpy(rng.uniform(-1, 1, (Co,)).astype(np.float32)).cuda()
        conv = wf.FoldedConv2d(w, b, x.shape, stride=s, padding=p, dtype=dt)
        y = conv(x).float().cpu().numpy()
        for i in (0, 5):
            ref = oracle.conv_padded(x[i:i + 1].float().cpu().numpy(), w.float().cpu().numpy(), b.cpu().numpy(), s, p)
            assert normrel(y[i:i + 1], ref) <= 1e-2


def test_tf32_path_within_1e3(golden_configs):
    y, ref, dt, conv = _config_run(golden_configs, "r50_b1", "")
    assert dt == "f32" and conv.device_plan["f"] % 2 == 0  # fold factor multiple of the stride
    assert normrel(y, ref) <= 1e-3
    y2 = wf.conv2d(golden_configs["r50_b1_x"], golden_configs["r50_b1_w"], 2, 2, padding=3,
                   bias=golden_configs["r50_b1_b"], precision="tf32")
    assert normrel(y2, ref) <= 1e-3


def test_grouped_conv_and_block_diagonal_check(oracle):
    rng = np.random.default_rng(4)
    x = rng.standard_normal((1, 10, 8, 1)).astype(np.float32)
    w = rng.standard_normal((3, 1, 1, 1)).astype(np.float32)
    x_f = wf.fold_input(x, 8)
    w_f = wf.expand_filter(w, 8)
    np.testing.assert_array_equal(wf.grouped_conv(x_f, w_f, 8), wf.conv2d(x_f, w_f))
    np.testing.assert_array_equal(wf.grouped_conv(x_f, w_f, 8), oracle.grouped_conv(x_f, w_f, 8))
    bad = w_f.copy()
    bad[0, 0, 0, 3] = 1e-30
    with pytest.raises(wf.NotBlockDiagonalError):
        wf.grouped_conv(x_f, bad, 8)


def test_conv1d_and_gemm_routes(oracle):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((12, 9, 1)).astype(np.float32)
    k = rng.standard_normal(4).astype(np.float32)
    y = wf.conv1d_h(x, k, 0.5)
    ref = oracle.bias_add(oracle.conv2d(x.reshape(1, 12, 9, 1), k.reshape(4, 1, 1, 1)),
                          np.array([0.5], np.float32)).reshape(9, 9, 1)
    np.testing.assert_array_equal(y, ref)
    a = rng.integers(-4, 5, (16, 3)).astype(np.float32)
    bm = rng.integers(-4, 5, (3, 4)).astype(np.float32)
    want = (a.astype(np.float64) @ bm.astype(np.float64)).astype(np.float32)
    np.testing.assert_array_equal(wf.gemm_ref(a, bm), want)
    np.testing.assert_array_equal(wf.gemm_as_conv1x1(a, bm), want)
    np.testing.assert_array_equal(wf.fold_tall_skinny(a, bm, 8), want)


@pytest.mark.parametrize("M,K,N,F,prec", [(8192, 3, 64, 8, "bf16"), (8000, 3, 64, 8, "bf16"), (4096, 4, 64, 4, "bf16"),
                                           (2048, 8, 128, 2, "f16"), (4096, 3, 64, 4, "tf32"),
                                           (4096, 3, 32, 8, "bf16"), (1024, 16, 96, 1, "bf16")])
def test_tall_skinny_gemm_on_tensor_cores(M, K, N, F, prec):
    """fold_tall_skinny through the folded tcgen05 kernel (SURVEY 8.F-3,
    src/gemm.cpp:51-69): exact on integer data (fp32 out), within the
    precision's tolerance on real data; gemm_as_conv1x1 through the unfolded
    variant of the same kernel."""
    rng = np.random.default_rng(M + K + N)
    a = rng.integers(-4, 5, (M, K)).astype(np.float32)
    b = rng.integers(-4, 5, (K, N)).astype(np.float32)
    want = a.astype(np.float64) @ b.astype(np.float64)
    got = wf.fold_tall_skinny(a, b, F, precision=prec, out_dtype=torch.float32)
    np.testing.assert_array_equal(got, want)
    a = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    b = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    dt = {"bf16": torch.bfloat16, "f16": torch.float16, "tf32": torch.float32}[prec]
    aq, bq = (torch.from_numpy(v).to(dt).float().numpy().astype(np.float64) for v in (a, b))
    got = wf.fold_tall_skinny(cuda(a, dt), cuda(b, dt), F, precision=prec)
    assert got.is_cuda and tuple(got.shape) == (M, N)
    assert normrel(got.float().cpu().numpy(), aq @ bq) <= (1e-3 if prec == "tf32" else 1e-2)
    if prec != "tf32" and N % 32 == 0:
        got = wf.gemm_as_conv1x1(a, b, precision=prec, out_dtype=torch.float32)
        assert normrel(got, aq @ bq) <= 1e-2


@pytest.mark.parametrize("geom", [(7, 64, 2, 3, 40), (3, 64, 1, 1, 32), (11, 96, 4, 0, 67), (3, 32, 2, 1, 32)],
                         ids=["r50", "vgg", "alexnet", "mnv2"])
def test_zero_padded_cin8_variant_exact(oracle, geom):
    """The zero-pad Cin 3 -> 8 comparison variant (the north star's baseline)
    equals the Cin = 3 oracle on integer data; AlexNet's (B = 190 KB) runs on
    CTA pairs, each SM holding half of B."""
    K, Co, s, p, hw = geom
    rng = np.random.default_rng(K * 100 + Co)
    x = rng.integers(-4, 5, (3, hw, hw, 3)).astype(np.float32)
    w = rng.integers(-4, 5, (K, K, 3, Co)).astype(np.float32)
    x8 = np.zeros((3, hw, hw, 8), np.float32)
    x8[..., :3] = x
    w8 = np.zeros((K, K, 8, Co), np.float32)
    w8[:, :, :3] = w
    conv = wf.FoldedConv2d(cuda(w8, torch.bfloat16), None, x8.shape, stride=s, padding=p, dtype=torch.bfloat16)
    y = conv(cuda(x8, torch.bfloat16), out_dtype=torch.float32)
    np.testing.assert_array_equal(y.cpu().numpy(), oracle.conv_padded(x, w, None, s, p))
    if K == 11:
        assert conv.device_plan["cta_pair"] == 2


def test_cuda_graph_replay_matches_eager():
    """FoldedConv2d.graphed(): the captured launch replays on new input contents."""
    torch.manual_seed(0)
    w = (torch.randn(7, 7, 3, 64, device="cuda") * 0.1).bfloat16()
    b = torch.randn(64, device="cuda")
    x = torch.randn(2, 64, 64, 3, device="cuda").bfloat16()
    conv = wf.FoldedConv2d(w, b, x.shape, stride=2, padding=3)
    replay, out = conv.graphed(x)
    for _ in range(2):
        x.copy_(torch.randn_like(x, dtype=torch.float32).bfloat16())
        replay()
        torch.testing.assert_close(out, conv(x), rtol=0, atol=0)


def test_sharded_launcher_single_rank():
    """shard.ShardedConv (the batch-sharded launcher) at world size 1 is the plain folded conv."""
    from paper_2601_11608_b200 import shard
    torch.manual_seed(3)
    w = (torch.randn(7, 7, 3, 64) * 0.1).bfloat16()
    b = torch.randn(64)
    x = torch.randn(5, 64, 64, 3).bfloat16()
    sc = shard.ShardedConv(w, b, x.shape, stride=2, padding=3)
    assert (sc.lo, sc.hi) == (0, 5)
    y = sc(x.cuda())
    ref = wf.FoldedConv2d(w.cuda(), b.cuda(), x.shape, stride=2, padding=3)(x.cuda())
    torch.testing.assert_close(sc.gather(y), ref, rtol=0, atol=0)


def test_no_cpu_fallback_on_cpu_tensors():
    conv = wf.FoldedConv2d(torch.randn(3, 3, 3, 16, device="cuda").bfloat16(), None, (1, 32, 32, 3), padding=1)
    with pytest.raises(ValueError):
        conv(torch.randn(1, 32, 32, 3).bfloat16())


@pytest.mark.parametrize("name", [n for n in CONFIG_GEOM if n != "r50_b1"])
def test_unfolded_variant_configs(golden_configs, name):
    """The same tcgen05 kernel on the UNFOLDED input (explicit im2col A tiles)."""
    y, ref, dt, conv = _config_run(golden_configs, name, "", variant="unfolded")
    assert conv.device_plan["producer"] == "im2col"
    assert normrel(y, ref) <= TOL[dt], name
    y, ref, _, _ = _config_run(golden_configs, name, "i", out_dtype=torch.float32, variant="unfolded")
    np.testing.assert_array_equal(y, ref, err_msg=name)


@pytest.mark.parametrize("kpair", ["0", "1"])
@pytest.mark.parametrize("name", [n for n in CONFIG_GEOM if n != "r50_b1"])
def test_gather_producer_matches_tma_bitwise(golden_configs, name, kpair, monkeypatch):
    """The software-gather producer builds the same shared-memory A image as the TMA boxes."""
    monkeypatch.setenv("WF_KPAIR", kpair)
    y0, _, _, conv = _config_run(golden_configs, name, "")
    assert conv.device_plan["producer"] in ("tma", "repitch+tma", "ring+tma", "gather")
    y1, _, _, _ = _config_run(golden_configs, name, "", flags=0x4000)
    np.testing.assert_array_equal(y0, y1)


def test_alexnet_full_geometry_sampled(oracle):
    """227x227 (1362-byte rows, partial last folded pixel, OW=55 masked tail), batch 5."""
    rng = np.random.default_rng(77)
    x = torch.from_numpy(rng.uniform(-1, 1, (5, 227, 227, 3)).astype(np.float32)).cuda().bfloat16()
    w = torch.from_numpy((rng.uniform(-1, 1, (11, 11, 3, 96)) / 18).astype(np.float32)).cuda().bfloat16()
    b = torch.from_numpy(rng.uniform(-1, 1, (96,)).astype(np.float32)).cuda()
    conv = wf.FoldedConv2d(w, b, x.shape, stride=4, padding=0, dtype=torch.bfloat16)
    assert conv.device_plan["producer"] == "repitch+tma"
    y = conv(x).float().cpu().numpy()
    y_gather = conv._forward(x, flags=A.WF_EPI_ROW_PRODUCER).float().cpu().numpy()  # row producer straight from x
    np.testing.assert_array_equal(y, y_gather)
    assert y.shape == (5, 55, 55, 96)
    for i in (0, 4):
        ref = oracle.conv_padded(x[i:i + 1].float().cpu().numpy(), w.float().cpu().numpy(), b.cpu().numpy(), 4, 0)
        assert normrel(y[i:i + 1], ref) <= 1e-2
    yu = wf.FoldedConv2d(w, b, x.shape, stride=4, padding=0, dtype=torch.bfloat16, variant="unfolded")(x)
    assert normrel(yu.float().cpu().numpy(), y) <= 1e-2


def test_unfolded_full_size_sampled(oracle):
    rng = np.random.default_rng(12)
    x = torch.from_numpy(rng.uniform(-1, 1, (3, 224, 224, 3)).astype(np.float32)).cuda().bfloat16()
    w = torch.from_numpy((rng.uniform(-1, 1, (7, 7, 3, 64)) / 12).astype(np.float32)).cuda().bfloat16()
    b = torch.from_numpy(rng.uniform(-1, 1, (64,)).astype(np.float32)).cuda()
    y = wf.FoldedConv2d(w, b, x.shape, stride=2, padding=3, variant="unfolded")(x).float().cpu().numpy()
    ref = oracle.conv_padded(x[2:3].float().cpu().numpy(), w.float().cpu().numpy(), b.cpu().numpy(), 2, 3)
    assert normrel(y[2:3], ref) <= 1e-2


def _random_device_geoms(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        s = int(rng.choice([1, 2, 4]))
        k = int(rng.integers(1, 12))
        p = int(rng.integers(0, min(4, k)))
        cout = int(rng.choice([32, 64, 96, 128]))
        dt = str(rng.choice(["bf16", "f16", "tf32"]))
        h = int(rng.integers(max(k, 4), 72))
        w = int(rng.integers(max(k, 8), 96))  # any width: W % f != 0 and odd pitches take the re-pitch path
        if w + 2 * p < k or h + 2 * p < k:
            continue
        out.append((k, cout, s, p, h, w, dt, int(rng.integers(1, 4))))
    return out


@pytest.mark.parametrize("geom", _random_device_geoms(40, 7), ids=lambda g: "k{}c{}s{}p{}h{}w{}{}n{}".format(*g))
def test_random_geometries_exact(oracle, geom):
    """Random first-layer geometries through the device kernel: bit-exact on integer data (fp32 out)."""
    K, Co, s, p, h, w, dt, n = geom
    tdt = {"bf16": torch.bfloat16, "f16": torch.float16, "tf32": torch.float32}[dt]
    rng = np.random.default_rng(K * 7919 + h * 31 + w)
    x = rng.integers(-3, 4, (n, h, w, 3)).astype(np.float32)
    wt = rng.integers(-3, 4, (K, K, 3, Co)).astype(np.float32)
    try:
        conv = wf.FoldedConv2d(cuda(wt, tdt), None, x.shape, stride=s, padding=p, dtype=tdt)
    except wf.UnsupportedError as e:
        pytest.skip(f"fold not applicable: {e}")
    y = conv(cuda(x, tdt), out_dtype=torch.float32)
    np.testing.assert_array_equal(y.cpu().numpy(), oracle.conv_padded(x, wt, None, s, p),
                                  err_msg=str(conv.device_plan))


def test_reference_acceptance_sweep_on_device():
    """The reference's oracle-equivalence sweep (tests/acceptance/acceptance_main.cpp:92-124):
    F in {1,2,4,8}, K in {1,2,3}, H in [K,8], W in {F,2F}, Cout in {1,2}; every
    case legal, apply_width_fold -> folded conv -> bias_add -> reconstruct on
    the device equals the unfolded conv + bias exactly (integer data)."""
    rng = np.random.default_rng(1002)
    cases = 0
    for F in (1, 2, 4, 8):
        for K in (1, 2, 3):
            for H in range(K, 9):
                for W in (F, 2 * F):
                    for Co in (1, 2):
                        x = rng.integers(-4, 5, (1, H, W, 1)).astype(np.float32)
                        w = rng.integers(-4, 5, (K, 1, 1, Co)).astype(np.float32)
                        b = rng.integers(-4, 5, (Co,)).astype(np.float32)
                        plan, x_f, w_f, b_f = wf.apply_width_fold(x, w, b, F)
                        assert plan["status"] == "apply", plan
                        y_f = wf.bias_add(wf.conv2d(x_f, w_f), b_f)
                        got = wf.reconstruct_output(y_f, F)
                        want = wf.bias_add(wf.conv2d(x, w), b)
                        np.testing.assert_array_equal(got, want, err_msg=f"F={F} K={K} H={H} W={W} Co={Co}")
                        cases += 1
    assert cases == 336


@pytest.mark.parametrize("n,h,k,co,s,p", [(64, 227, 11, 96, 4, 0), (7, 227, 11, 96, 4, 0), (16, 224, 3, 64, 1, 1)])
def test_multicast_cluster_matches_single_cta(monkeypatch, n, h, k, co, s, p):
    """Two-N-tile plans can run as a 2-CTA cluster sharing A stages by TMA multicast
    (opt-in WF_MCAST=1, read at plan time) instead of one CTA per N-tile (the
    default, WF_MCAST=0 forces it). Bit-identical."""
    torch.manual_seed(5)
    x = torch.randn(n, h, h, 3, device="cuda").to(torch.bfloat16)
    w = (torch.randn(k, k, 3, co, device="cuda") * 0.1).to(torch.bfloat16)
    b = torch.randn(co, device="cuda")
    monkeypatch.setenv("WF_MCAST", "1")
    conv = wf.FoldedConv2d(w, b, x.shape, stride=s, padding=p, dtype=torch.bfloat16)
    assert conv.device_plan["n_tiles"] == 2 and conv.device_plan["launch_opts"] & 16
    y_mc = conv(x)
    monkeypatch.setenv("WF_MCAST", "0")
    conv_one = wf.FoldedConv2d(w, b, x.shape, stride=s, padding=p, dtype=torch.bfloat16)
    assert conv_one.device_plan["launch_opts"] & 8
    y_one = conv_one(x)
    torch.cuda.synchronize()
    assert torch.equal(y_mc, y_one)
    ref = torch.nn.functional.conv2d(x.float().permute(0, 3, 1, 2), w.float().permute(3, 2, 0, 1), b, stride=s,
                                     padding=p).permute(0, 2, 3, 1)
    assert ((y_mc.float() - ref).norm() / ref.norm()).item() < 1e-2
