"""CPU replay of the tcgen05 schedule (no GPU): every MMA of an M tile is
re-executed in numpy from the planner's own description (wf_schedule_describe)
-- A rows read through the descriptor addressing (start address + row * 16 B,
core column 1 at +LBO; SWIZZLE_32B: 32-byte rows) out of the A-stage layout the
TMA boxes land, B built from the per-core-column (kh, c, slot mask) words and
the generalized expansion -- and the accumulators, mapped through the slot
order and the epilogue's column permutation, must equal the oracle conv
bit-exactly on integer data. This pins the planner (both K-step schedules,
zero-init order, half-split reorder) independently of the device.
"""
import numpy as np
import pytest

from paper_2601_11608_b200 import _abi as A

DT = {"bf16": A.WF_BF16, "f16": A.WF_F16, "tf32": A.WF_TF32}


def chunk_perm(col, ch):
    c, w = col // ch, col % ch
    return c * ch + (ch // 4) * ((w % 8) // 2) + 2 * (w // 8) + (w % 2)


def replay(oracle, x, w, s, p, dtype, n_img=None):
    N, H, W, C = x.shape
    KH, KW, _, Co = w.shape
    d = A.make_desc(N, H, W, C, KH, KW, Co, s, s, p, p)
    sc = A.schedule_describe(d, 0, 0, DT[dtype])
    f, r, c0, kwf = sc["f"], sc["r"], sc["c0"], sc["kw_f"]
    esz = sc["esize"]
    E2 = 16 // esz  # elements per 16-byte core column
    Wbox, OHt, tps = sc["wbox"], sc["tile_rows"], sc["tps"]
    Ng, CH = sc["Ng"], sc["CH"]
    OH, OW = (H + 2 * p - KH) // s + 1, (W + 2 * p - KW) // s + 1
    Wfo = -(-OW // r)
    wexp = oracle.expand_filter_folded(w, f, s, p).astype(np.float64)  # (KH, KW', f*C, r*Co)
    yref = oracle.conv_padded(x, w, None, s, p).astype(np.float64)
    ent = np.array(sc["entries"], np.int64).reshape(-1, 7)
    nt = np.array(sc["ntiles"], np.int64).reshape(-1, 6)
    order = sc["order"]
    amin = sc["amin"]
    xd = x.astype(np.float64)

    def a_rows(n, oh0, addr):
        """Elements of core column(s) at byte addresses `addr` (one per M row) of the A stage."""
        out = np.zeros((len(addr), E2))
        # rows whose view runs past the stage (columns w >= Wfo of the last
        # row, discarded by the epilogue) read padding: NaN marks them here
        past = addr >= sc["stage_bytes"]
        out[past] = np.nan
        addr = np.where(past, 0, addr)
        if sc["sw32"]:
            b, rem = addr // sc["region_bytes"], addr % sc["region_bytes"]
            qi, rem2 = rem // sc["qregion_bytes"], rem % sc["qregion_bytes"]
            pos, half = rem2 // 32, (rem2 % 32) // 16
            q = np.array(sc["qs"])[qi] + half
        else:
            b, rem = addr // sc["region_bytes"], addr % sc["region_bytes"]
            q, rem2 = rem // sc["lbo_a"], rem % sc["lbo_a"]
            assert (rem2 % 16 == 0).all()
            pos = rem2 // 16
        i, wcol = pos // Wbox, pos % Wbox
        am = np.array(amin)[b]
        assert (am[~past] != -999).all(), "A view in a residue without filter rows"
        ih = (oh0 + am + i) * s + b
        for e in range(E2):
            k = q * E2 + e  # region q == Q (the shift region) is core column 0 of the next folded pixel
            kin = k % (f * C)
            iw = (c0 + wcol + k // (f * C)) * f + kin // C
            ch = kin % C
            ok = (ih >= 0) & (ih < H) & (iw >= 0) & (iw < W) & ~past
            out[ok, e] = xd[n, ih[ok], iw[ok], ch[ok]]
        return out

    m = np.arange(128)
    checked = 0
    for ti in range(len(nt)):
        col0, cols, e0, ne, g0, split = nt[ti]
        for n in range(N if n_img is None else n_img):
            for oh_t in range(0, OH, OHt):
                k_in_stage = (oh_t // OHt) % tps
                oh_stage = oh_t - k_in_stage * OHt
                D = np.zeros((128, cols))
                for a_off, lbo, b_off, meta, tcol, w0, w1 in ent[e0:e0 + ne]:
                    Nm = ((meta >> 22) & 0x1FF) * 8
                    slot0 = (meta >> 16) & 0x3F
                    accf = (meta >> 31) & 1
                    base = a_off + k_in_stage * sc["tile_shift"]
                    if sc["sw32"]:
                        A0 = a_rows(n, oh_stage, base + m * 32)
                        A1 = a_rows(n, oh_stage, base + m * 32 + 16)
                    else:
                        A0 = a_rows(n, oh_stage, base + m * 16)
                        A1 = a_rows(n, oh_stage, base + lbo + m * 16)
                    Bm = np.zeros((2, Nm, E2))
                    for cc, word in enumerate((w0, w1)):
                        kh, c, mask = word & 0xFF, (word >> 8) & 0xFF, word >> 16
                        widx = c * E2 + np.arange(E2)
                        kp, kk = widx // (f * C), widx % (f * C)
                        for nn in range(Nm):
                            sl = slot0 + nn // Ng
                            if not (mask >> (nn // Ng)) & 1:
                                continue
                            ocol = order[g0 + sl] * Ng + chunk_perm(nn % Ng, CH)
                            okk = kp < kwf
                            Bm[cc, nn, okk] = wexp[kh, kp[okk], kk[okk], ocol]
                    prod = A0 @ Bm[0].T + A1 @ Bm[1].T
                    if accf:
                        D[:, tcol:tcol + Nm] += prod
                    else:
                        D[:, tcol:tcol + Nm] = prod
                for col in range(cols):
                    g = order[g0 + col // Ng]
                    ocol = g * Ng + chunk_perm(col % Ng, CH)
                    j, co = ocol // Co, ocol % Co
                    t, wq = m // Wbox, m % Wbox
                    oh, ow = oh_t + t, wq * r + j
                    ok = (wq < Wfo) & (t < OHt) & (oh < OH) & (ow < OW)
                    np.testing.assert_array_equal(D[ok, col], yref[n, oh[ok], ow[ok], co],
                                                  err_msg=f"tile oh0={oh_t} n={n} col={col}")
                    checked += int(ok.sum())
    assert checked > 0
    return sc


GEOMS = [  # (KH, KW, Cout, stride, pad, H, W, dtype)
    (7, 7, 64, 2, 3, 24, 32, "bf16"),     # R50 conv1
    (3, 3, 64, 1, 1, 12, 32, "bf16"),     # VGG16 conv1_1
    (11, 11, 96, 4, 0, 27, 35, "bf16"),   # AlexNet conv1 (W % f != 0)
    (3, 3, 32, 2, 1, 16, 32, "f16"),      # MobileNetV2 stem
    (7, 7, 64, 2, 3, 16, 32, "tf32"),     # R50 conv1, TF32 (f = 4)
    (1, 1, 64, 1, 0, 300, 8, "bf16"),     # tall-skinny GEMM (M=2400, K=3, N=64) as a folded 1x1 conv
]


@pytest.mark.parametrize("tps", ["", "2", "4"])
@pytest.mark.parametrize("kpair", ["0", "1"])
@pytest.mark.parametrize("geom", GEOMS, ids=["r50", "vgg", "alexnet", "mnv2", "r50_tf32", "gemm"])
def test_schedule_replay_exact(oracle, monkeypatch, geom, kpair, tps):
    monkeypatch.setenv("WF_KPAIR", kpair)
    if tps:
        monkeypatch.setenv("WF_TPS", tps)  # M tiles per A stage (the batch here is too small to pick them)
    KH, KW, Co, s, p, H, W, dt = geom
    rng = np.random.default_rng(KH * 7 + W)
    x = rng.integers(-3, 4, (1, H, W, 3)).astype(np.float32)
    w = rng.integers(-3, 4, (KH, KW, 3, Co)).astype(np.float32)
    sc = replay(oracle, x, w, s, p, dt)
    assert bool(sc["kpair"]) == (kpair == "1")


def _random_geoms(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        s = int(rng.choice([1, 2, 4]))
        k = int(rng.integers(1, 12))
        p = int(rng.integers(0, min(4, k)))
        cout = int(rng.choice([32, 64, 96, 128]))
        dt = str(rng.choice(["bf16", "f16", "tf32"]))
        h = int(rng.integers(max(k, 4), 40))
        w = int(rng.choice([8, 16, 24, 32, 48, 64]))
        if w + 2 * p < k or h + 2 * p < k:
            continue
        out.append((k, k, cout, s, p, h, w, dt))
    return out


@pytest.mark.parametrize("geom", _random_geoms(24, 2024), ids=lambda g: "k{}s{}p{}c{}h{}w{}{}".format(
    g[0], g[3], g[4], g[2], g[5], g[6], g[7]))
def test_schedule_replay_random_geometries(oracle, geom):
    """Random kernels / strides / paddings / widths / dtypes: whatever the
    planner builds (or falls back from) replays exactly."""
    KH, KW, Co, s, p, H, W, dt = geom
    N, Hh, Ww = 1, H, W
    d = A.make_desc(N, Hh, Ww, 3, KH, KW, Co, s, s, p, p)
    plan = A.plan_fold(d, 0, 0, DT[dt])
    if plan.status != A.WF_FOLD_APPLY:
        pytest.skip(f"fold falls back: {A.REASONS[plan.reason]}")
    rng = np.random.default_rng(KH * 1000 + W)
    x = rng.integers(-3, 4, (N, Hh, Ww, 3)).astype(np.float32)
    w = rng.integers(-3, 4, (KH, KW, 3, Co)).astype(np.float32)
    replay(oracle, x, w, s, p, dt)


@pytest.mark.parametrize("geom", [(1, 1, 64, 1, 0, 47, 32, 4, "bf16"), (1, 1, 32, 1, 0, 12, 16, 8, "f16"),
                                  (3, 3, 64, 1, 1, 20, 16, 8, "bf16"), (5, 5, 96, 2, 2, 24, 32, 4, "bf16"),
                                  (1, 1, 64, 2, 0, 16, 32, 2, "tf32"), (3, 3, 32, 1, 1, 14, 24, 2, "bf16")],
                         ids=lambda g: "k{}s{}p{}c{}C{}{}".format(g[0], g[3], g[4], g[2], g[7], g[8]))
def test_schedule_replay_other_channel_counts(oracle, geom):
    """Cin != 3, including one-core-column window rows (a 1x1 conv on 16-byte folded pixels): every MMA
    of a valid output row reads only loaded A (the replay marks unloaded bytes NaN; a zero-B partner
    column outside the window used to read past the stage -- found by the real-data GPU fuzz)."""
    KH, KW, Co, s, p, H, W, C, dt = geom
    d = A.make_desc(1, H, W, C, KH, KW, Co, s, s, p, p)
    plan = A.plan_fold(d, 0, 0, DT[dt])
    if plan.status != A.WF_FOLD_APPLY:
        pytest.skip(f"fold falls back: {A.REASONS[plan.reason]}")
    rng = np.random.default_rng(KH * 100 + W + C)
    x = rng.integers(-3, 4, (1, H, W, C)).astype(np.float32)
    w = rng.integers(-3, 4, (KH, KW, C, Co)).astype(np.float32)
    replay(oracle, x, w, s, p, dt)
