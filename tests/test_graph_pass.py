"""The rewrite-rule pass and the device interpreter.

CPU: pass decisions, value ids preserved, bias fusion, idempotence, shape
errors (the reference pass contract, include/widthfold/pass.hpp:45-52 and
acceptance_main.cpp:268-313). GPU: pass soundness on 100 random graphs --
the folded TF32 graph equals the unfolded exact-fp32 graph bit-for-bit on
integer data (every product and partial sum is exact) and within 1e-3
normwise on float data."""
import numpy as np
import pytest

import paper_2601_11608_b200 as wf
from tests.graphs import random_graph


def r50_graph(batch=2, hw=32):
    g = wf.Graph()
    g.add("x", "input", shape=[batch, hw, hw, 3])
    g.constant("w", np.ones((7, 7, 3, 64), np.float32))
    g.add("conv", "conv2d", ["x", "w"], stride_h=2, stride_w=2, pad_h=3, pad_w=3)
    g.constant("b", np.arange(64, dtype=np.float32))
    g.add("bias", "bias_add", ["conv", "b"])
    g.add("y", "output", ["bias"])
    return g


def test_pass_rewrites_r50_stem_and_fuses_the_bias():
    g, rep = wf.width_fold_pass(r50_graph())
    assert rep["applied_count"] == 1
    d = rep["decisions"][0]
    assert d["id"] == "conv" and d["applied"] and d["plan"]["factor"] == 4  # tf32: 48-byte folded pixel
    assert "bias folded via bias" in d["note"]
    conv = g.find("conv")
    assert conv["op"] == "folded_conv2d" and conv["bias"] and conv["inputs"] == ["x", "w", "b"]
    assert g.find("bias")["op"] == "reshape"  # the bias_add keeps its value id as a view
    assert g.find("y")["out_shape"] == [2, 16, 16, 64]
    assert rep["before"]["macs"] == rep["after"]["macs"] == 2 * 16 * 16 * 64 * 7 * 7 * 3
    assert not rep["before"]["aligned"] and rep["after"]["aligned"]


def test_pass_is_idempotent():
    g1, r1 = wf.width_fold_pass(r50_graph())
    g2, r2 = wf.width_fold_pass(g1)
    assert r2["applied_count"] == 0
    assert [d["plan"]["reason"] for d in r2["decisions"]] == ["AlreadyAligned"]
    assert g2.nodes == g1.nodes


def test_pass_skip_reasons():
    g = wf.Graph()
    g.add("x", "input", shape=[1, 8, 8, 8])
    g.constant("w8", np.ones((3, 3, 8, 16), np.float32))
    g.add("aligned", "conv2d", ["x", "w8"])
    g.add("xin", "input", shape=[3, 3, 8, 16])  # a non-constant filter
    g.add("dyn", "conv2d", ["x", "xin"])
    g.add("y0", "output", ["aligned"])
    g.add("y1", "output", ["dyn"])
    _, rep = wf.width_fold_pass(g)
    reasons = {d["id"]: d["plan"]["reason"] for d in rep["decisions"]}
    assert reasons == {"aligned": "AlreadyAligned", "dyn": "AlreadyAligned"}
    g3 = wf.Graph()
    g3.add("x", "input", shape=[1, 8, 8, 3])
    g3.add("xin", "input", shape=[3, 3, 3, 16])
    g3.add("dyn", "conv2d", ["x", "xin"])
    g3.add("y", "output", ["dyn"])
    _, rep3 = wf.width_fold_pass(g3)
    assert rep3["decisions"][0]["plan"]["reason"] == "NotProfitable"
    assert "not a constant" in rep3["decisions"][0]["note"]
    _, rep4 = wf.width_fold_pass(r50_graph(), factor=1)
    assert rep4["decisions"][0]["plan"]["reason"] == "AlreadyAligned"
    _, rep5 = wf.width_fold_pass(r50_graph(), factor=3)  # 3 is not a multiple of the W stride 2
    assert rep5["decisions"][0]["plan"]["reason"] == "StrideOnFoldAxis"


def test_pass_and_shape_errors():
    with pytest.raises(ValueError):
        wf.width_fold_pass(r50_graph(), align=0)
    bad = wf.Graph()
    bad.add("y", "output", ["x"])
    with pytest.raises(wf.ShapeInferenceFailureError):
        bad.infer_shapes()
    g = r50_graph()
    g.find("bias")["inputs"] = ["conv", "w"]  # a rank-4 "bias"
    with pytest.raises(wf.ShapeInferenceFailureError):
        wf.width_fold_pass(g)


@pytest.mark.parametrize("seed", range(0, 100, 7))
def test_random_graphs_rewrite_totally(seed):
    g, _ = random_graph(seed, integer=True)
    g2, rep = wf.width_fold_pass(g)
    assert len(rep["decisions"]) == sum(n["op"] == "conv2d" for n in g.nodes)
    ids = {n["id"] for n in g.nodes if n["op"] in ("output", "input")}
    assert ids <= {n["id"] for n in g2.nodes}  # value ids preserved
    before = {n["id"]: n["out_shape"] for n in g.infer_shapes().nodes if n["op"] == "output"}
    after = {n["id"]: n["out_shape"] for n in g2.nodes if n["op"] == "output"}
    assert before == after


@pytest.mark.gpu
def test_interpreter_runs_the_reference_semantics(oracle):
    g = r50_graph(batch=1, hw=24)
    rng = np.random.default_rng(3)
    x = rng.integers(-4, 5, (1, 24, 24, 3)).astype(np.float32)
    y = wf.interpret(g, {"x": x}, mode="dense")["y"]
    ref = oracle.conv_padded(x, np.ones((7, 7, 3, 64), np.float32), np.arange(64, dtype=np.float32), 2, 3)
    np.testing.assert_array_equal(y, ref)
    with pytest.raises(wf.MissingInputError):
        wf.interpret(g, {}, mode="dense")


@pytest.mark.gpu
def test_pass_soundness_on_random_graphs():
    """acceptance_main.cpp:268-313 on the device: 100 random graphs."""
    applied = 0
    for seed in range(100):
        integer = seed % 2 == 0
        g, inputs = random_graph(seed, integer)
        g2, rep = wf.width_fold_pass(g)
        applied += rep["applied_count"]
        y0 = wf.interpret(g, inputs, mode="dense")
        y1 = wf.interpret(g2, inputs, mode="device")
        assert y0.keys() == y1.keys()
        for k in y0:
            if integer:
                np.testing.assert_array_equal(y1[k], y0[k], err_msg=f"seed {seed} output {k}")
            else:
                err = np.max(np.abs(y1[k] - y0[k])) / max(np.max(np.abs(y0[k])), 1e-30)
                assert err <= 1e-3, (seed, k, err)
    assert applied >= 50  # most random first layers fold


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["bf16", "f16"])
def test_pass_at_16_bit_precision(precision, tmp_path):
    """width_fold_pass(precision=bf16/f16): folded nodes cast their f32 input and
    filter on the device; integer graphs stay exact (small integers are exact in
    16 bits), real-valued ones within 1e-2; the node dtype survives write/read."""
    applied = 0
    for seed in range(20):
        integer = seed % 2 == 0
        g, inputs = random_graph(seed, integer)
        g2, rep = wf.width_fold_pass(g, precision=precision)
        applied += rep["applied_count"]
        assert all(n.get("dtype") == precision for n in g2.nodes if n["op"] == "folded_conv2d")
        y0 = wf.interpret(g, inputs, mode="dense")
        y1 = wf.interpret(g2, inputs, mode="device")
        for k in y0:
            if integer:
                np.testing.assert_array_equal(y1[k], y0[k], err_msg=f"seed {seed} output {k}")
            else:
                err = np.max(np.abs(y1[k] - y0[k])) / max(np.max(np.abs(y0[k])), 1e-30)
                assert err <= 1e-2, (seed, k, err)
        if seed == 0:
            wf.write_graph(g2, tmp_path / "g.json")
            back = wf.read_graph(tmp_path / "g.json")
            assert [n.get("dtype") for n in back.nodes] == [n.get("dtype") for n in g2.nodes]
    assert applied >= 10
