"""CPU: pin the plain-C oracle (oracle/oracle.c) to the reference.

Every check is against golden vectors produced by the reference's own code
(tests/golden/make_golden.py) or, when it was compiled here, against the
reference library itself (oracle/_ref). Exact equality everywhere: the oracle
keeps the reference's reduction order and its no-FMA codegen.
"""
import ctypes
import os

import numpy as np
import pytest

from tests.conftest import ROOT

CONFIG_GEOM = {  # name -> fold factor the device uses (f % stride == 0, 32-byte folded pixel)
    "r50_b1": 4, "vgg16": 8, "alexnet": 8, "mnv2": 8, "r50_b8192": 8,
}


def test_conv_cases_bitwise(oracle, golden_conv):
    tags = sorted({k.rsplit("_", 1)[0] for k in golden_conv if k.endswith("_x")})
    assert len(tags) == 12
    for tag in tags:
        g = {k[len(tag) + 1:]: v for k, v in golden_conv.items() if k.startswith(tag + "_")}
        sh, sw = (int(v) for v in g["stride"])
        y = oracle.conv2d(g["x"], g["w"], sh, sw)
        np.testing.assert_array_equal(y.view(np.uint32), g["y"].view(np.uint32), err_msg=tag)
        np.testing.assert_array_equal(oracle.bias_add(y, g["b"]).view(np.uint32), g["yb"].view(np.uint32),
                                      err_msg=tag)


def test_appendix_a_pipeline(oracle, golden_appendix):
    for kind in ("float", "int"):
        g = {k[len(kind) + 1:]: v for k, v in golden_appendix.items() if k.startswith(kind + "_")}
        x_f = oracle.fold_input_general(g["x"], 8)
        w_f = oracle.expand_filter_general(g["w"], 8)
        b_f = oracle.replicate_bias(g["b"], 8)
        np.testing.assert_array_equal(x_f, g["x_f"])
        np.testing.assert_array_equal(w_f, g["w_f"])
        np.testing.assert_array_equal(b_f, g["b_f"])
        y = oracle.reconstruct_output(oracle.bias_add(oracle.conv2d(x_f, w_f), b_f), 8)
        np.testing.assert_array_equal(y, g["y_folded"])
        y_ref = oracle.bias_add(oracle.conv2d(g["x"], g["w"]), g["b"])
        np.testing.assert_array_equal(y_ref, g["y_ref"])
        if kind == "int":
            np.testing.assert_array_equal(y, y_ref)
        else:
            assert np.max(np.abs(y - y_ref)) <= 1e-5  # Appendix-A tolerance


def test_hand_kats(oracle, golden_kats):
    g = golden_kats
    np.testing.assert_array_equal(g["fold_4"].ravel(), [10, 11, 12, 13])
    np.testing.assert_array_equal(oracle.fold_input_general(g["fold_general_in"], 2), g["fold_general_out"])
    np.testing.assert_array_equal(oracle.expand_filter_general(g["expand_in"], 2), g["expand_out"])
    np.testing.assert_array_equal(oracle.replicate_bias(np.array([1, 2], np.float32), 3), g["replicate"])
    np.testing.assert_array_equal(oracle.expand_filter_general(g["expand_general_in"], 4), g["expand_general_out_f4"])
    assert list(g["mac_report"]) == [8960, 71680, 8960, 71680]
    assert oracle.count_macs(1, 28, 64, 1, 5, 1, 1) == 8960


def test_padded_configs_bitwise(oracle, golden_configs):
    for name in CONFIG_GEOM:
        KH, KW, C, Co, s, p, relu = (int(v) for v in golden_configs[f"{name}_geom"])
        for suffix in ("", "i"):
            x, w, b = (golden_configs[f"{name}_{k}{suffix}"] for k in ("x", "w", "b"))
            y = oracle.conv_padded(x, w, b, s, p, bool(relu))
            np.testing.assert_array_equal(y, golden_configs[f"{name}_y{suffix}"], err_msg=name + suffix)


@pytest.mark.parametrize("name", list(CONFIG_GEOM))
def test_generalized_fold_is_the_reference_conv(oracle, golden_configs, name):
    """Appendix-A expansion + folded evaluation == reference conv2d of the padded input.

    Integer data: exact. Float data: equal up to the sign of zero,
    because skipped taps are exact zero products and the surviving terms keep
    the reference's kh -> kw -> ci order.
    """
    KH, KW, C, Co, s, p, relu = (int(v) for v in golden_configs[f"{name}_geom"])
    f = CONFIG_GEOM[name]
    for suffix in ("i", ""):
        x, w, b = (golden_configs[f"{name}_{k}{suffix}"] for k in ("x", "w", "b"))
        wexp = oracle.expand_filter_folded(w, f, s, p)
        y = oracle.conv_folded(x, wexp, KH, KW, Co, f, s, p, p)
        y = oracle.bias_add(y, b)
        if relu:
            y = oracle.relu(y)
        np.testing.assert_array_equal(y, golden_configs[f"{name}_y{suffix}"], err_msg=name + suffix)


def test_generalized_expansion_reduces_to_reference(oracle, golden_kats):
    w = golden_kats["expand_general_in"]
    np.testing.assert_array_equal(oracle.expand_filter_folded(w, 4, 1, 0), golden_kats["expand_general_out_f4"])


def test_fold_geometry_formulas(oracle):
    # SURVEY.md section 8 folded-view table
    assert oracle.fold_geometry(8, 2, 3, 7) == (4, -1, 3)     # R50 f=8
    assert oracle.fold_geometry(16, 2, 3, 7) == (8, -1, 3)    # R50 f=16 ("Cout=512")
    assert oracle.fold_geometry(8, 1, 1, 3) == (8, -1, 3)     # VGG16
    assert oracle.fold_geometry(8, 4, 0, 11) == (2, 0, 2)     # AlexNet
    assert oracle.fold_geometry(8, 2, 1, 3) == (4, -1, 2)     # MNv2
    assert oracle.fold_geometry(4, 2, 3, 7) == (2, -1, 3)     # R50 b1 fp32 f=4


def test_fold_is_a_reshape_and_bijective(oracle):
    rng = np.random.default_rng(1003)
    for _ in range(200):
        F = int(rng.integers(1, 9))
        B, H, C = int(rng.integers(1, 3)), int(rng.integers(1, 9)), int(rng.integers(1, 5))
        W = F * int(rng.integers(1, 7))
        x = rng.uniform(-1, 1, (B, H, W, C)).astype(np.float32)
        xf = oracle.fold_input_general(x, F)
        np.testing.assert_array_equal(xf, x.reshape(B, H, W // F, F * C))
        np.testing.assert_array_equal(oracle.unfold_input_general(xf, F), x)
        np.testing.assert_array_equal(oracle.reconstruct_output(xf, F), x)


def test_grouped_equals_dense_bitwise(oracle):
    rng = np.random.default_rng(1005)
    for F in (1, 2, 4, 8):
        for K in (1, 2, 3):
            x = rng.integers(-4, 5, (1, 8, 2 * F, 1)).astype(np.float32)
            w = rng.uniform(-1, 1, (K, 1, 1, 2)).astype(np.float32)
            xf = oracle.fold_input_general(x, F)
            wf = oracle.expand_filter_general(w, F)
            np.testing.assert_array_equal(oracle.grouped_conv(xf, wf, F), oracle.conv2d(xf, wf))


REF_SO = os.path.join(ROOT, "oracle", "_ref", "libwidthfold_ref.so")


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference library not built here")
def test_oracle_matches_reference_library(oracle):
    lib = ctypes.CDLL(REF_SO)
    fp = ctypes.POINTER(ctypes.c_float)
    i64 = ctypes.c_int64
    rng = np.random.default_rng(11)
    for _ in range(30):
        B, H, W, C = (int(v) for v in rng.integers(1, 4, 1).tolist() + rng.integers(5, 14, 2).tolist()
                      + rng.integers(1, 5, 1).tolist())
        KH, KW = int(rng.integers(1, 6)), int(rng.integers(1, 6))
        Co, sh, sw = int(rng.integers(1, 9)), int(rng.integers(1, 4)), int(rng.integers(1, 4))
        x = rng.uniform(-1, 1, (B, H, W, C)).astype(np.float32)
        w = rng.uniform(-1, 1, (KH, KW, C, Co)).astype(np.float32)
        b = rng.uniform(-1, 1, (Co,)).astype(np.float32)
        want = oracle.bias_add(oracle.conv2d(x, w, sh, sw), b)
        got = np.empty_like(want)
        rc = lib.wfref_conv2d(x.ctypes.data_as(fp), i64(B), i64(H), i64(W), i64(C), w.ctypes.data_as(fp), i64(KH),
                              i64(KW), i64(Co), i64(sh), i64(sw), b.ctypes.data_as(fp), 0, got.ctypes.data_as(fp))
        assert rc == 0
        np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))
