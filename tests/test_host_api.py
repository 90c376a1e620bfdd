"""CPU: the C++ host layer (_core, namespace widthfold) reproduces the
reference's host-side API: legality, auto factor, MAC accounting, errors."""
import ast

import numpy as np
import pytest

import paper_2601_11608_b200 as wf
from paper_2601_11608_b200 import _core


def test_reference_names_exported():
    ref_names = ["apply_width_fold", "apply_width_fold_general", "bias_add", "check_legality",
                 "choose_fold_factor", "conv1d_h", "conv2d", "count_macs", "expand_filter",
                 "expand_filter_general", "fold_input", "fold_input_general", "fold_tall_skinny",
                 "gemm_as_conv1x1", "gemm_ref", "grouped_conv", "mac_report", "reconstruct_output",
                 "replicate_bias", "unfold_input_general"]  # /root/reference/proj/python/widthfold/__init__.py:27-48
    for n in ref_names:
        assert callable(getattr(wf, n)), n
        assert n in wf.__all__


def test_exception_hierarchy():
    assert issubclass(wf.ShapeMismatchError, ValueError)
    assert issubclass(wf.IllegalFoldError, ValueError)
    assert issubclass(wf.DegenerateOutputError, ValueError)
    assert issubclass(wf.NotBlockDiagonalError, RuntimeError)


def test_legality_table_matches_reference(golden_kats):
    for row in golden_kats["legality"]:
        shape, filt, f, status, reason, fis, efs = ast.literal_eval(str(row))
        p = wf.check_legality(shape, filt, f)
        assert (p["status"], p["reason"], p["folded_input_shape"], p["expanded_filter_shape"]) == \
            (status, reason, fis, efs), row


def test_choose_table_matches_reference(golden_kats):
    for row in golden_kats["choose"]:
        shape, filt, status, reason, factor, fis, efs = ast.literal_eval(str(row))
        p = wf.choose_fold_factor(shape, filt)
        assert (p["status"], p["reason"], p["factor"], p["folded_input_shape"], p["expanded_filter_shape"]) == \
            (status, reason, factor, fis, efs), row


def test_mac_report_and_count_macs(golden_kats):
    r = wf.mac_report([1, 32, 64, 1], [5, 1, 1, 1], 8)
    assert [r["original"], r["dense_folded"], r["grouped_folded"], r["zero_padded"]] == \
        list(golden_kats["mac_report"])
    r = wf.mac_report([1, 16, 16, 3], [3, 1, 3, 4], 8)
    assert [r["original"], r["dense_folded"], r["grouped_folded"], r["zero_padded"]] == \
        list(golden_kats["mac_report_rgb"])
    assert wf.count_macs([1, 32, 64, 1], [5, 1, 1, 1]) == golden_kats["count_macs"][0]
    assert wf.count_macs([2, 9, 11, 3], [3, 2, 3, 5], 2, 3) == golden_kats["count_macs"][1]
    with pytest.raises(ValueError):
        wf.mac_report([1, 4, 7, 1], [3, 1, 1, 1], 8)  # fallback plan -> invalid_argument


def test_errors_match_reference():
    with pytest.raises(wf.ShapeMismatchError):
        wf.check_legality([1, 8, 8], [3, 1, 1, 1], 2)
    with pytest.raises(wf.DegenerateOutputError):
        wf.check_legality([1, 2, 8, 1], [3, 1, 1, 1], 2)
    with pytest.raises(ValueError):
        wf.check_legality([1, 8, 8, 1], [3, 1, 1, 1], 0)
    with pytest.raises(ValueError):
        wf.choose_fold_factor([1, 8, 8, 1], [3, 1, 1, 1], align=0)


CONFIGS = {  # name: (input, filter, stride, pad, dtype) -- BASELINE.json configs
    "r50_b1": ([1, 224, 224, 3], [7, 7, 3, 64], 2, 3, "tf32"),
    "vgg16": ([256, 224, 224, 3], [3, 3, 3, 64], 1, 1, "bf16"),
    "mnv2": ([1024, 224, 224, 3], [3, 3, 3, 32], 2, 1, "f16"),
    "r50_b8192": ([8192, 224, 224, 3], [7, 7, 3, 64], 2, 3, "bf16"),
    "alexnet": ([512, 227, 227, 3], [11, 11, 3, 96], 4, 0, "bf16"),
}


@pytest.mark.parametrize("name", list(CONFIGS))
def test_device_plans_for_configs(name, oracle):
    shape, filt, s, p, dt = CONFIGS[name]
    plan = wf.plan_fold(shape, filt, s, s, p, p, dtype=dt)
    assert plan["status"] == "apply", plan
    d = plan["device"]
    esize = 4 if dt == "tf32" else 2
    assert d["f"] % s == 0 and (d["f"] * 3 * esize) % 16 == 0
    r, c0, kwf = oracle.fold_geometry(d["f"], s, p, filt[1])
    assert (d["r"], d["c0"], d["kw_f"]) == (r, c0, kwf)
    assert plan["expanded_filter_shape"] == [filt[0], kwf, d["f"] * 3, r * filt[3]]
    oh = (shape[1] + 2 * p - filt[0]) // s + 1
    assert d["producer"] == ("repitch+tma" if name == "alexnet" else "tma")
    assert d["useful_macs"] == wf.count_macs(shape, filt, s, s, p, p)
    assert d["useful_macs"] == shape[0] * oh * oh * filt[3] * filt[0] * filt[1] * 3
    assert d["issued_macs"] >= d["useful_macs"]


def test_alexnet_plan_repitches_or_gathers_unaligned_rows(monkeypatch):
    # W = 227 is prime: no pure-reshape fold exists (the reference says WidthNotDivisible,
    # src/fold.cpp:58) and the 1362-byte row pitch cannot be a TMA stride, so the
    # generalized fold re-pitches x into a 232-pixel workspace (zero tail) on the
    # device, then runs the TMA path with a masked output tail (OW = 55, r = 2).
    plan = wf.plan_fold([512, 227, 227, 3], [11, 11, 3, 96], 4, 4, 0, 0, dtype="bf16")
    assert plan["status"] == "apply", plan
    d = plan["device"]
    assert (d["f"], d["r"], d["producer"]) == (8, 2, "repitch+tma")
    assert d["pitched_w"] == 232 and d["workspace_bytes"] == 512 * 227 * 232 * 3 * 2
    assert d["wf"] == 29 and d["wfo"] == 28 and d["ow"] == 55
    # WF_RING=1 (producer 5): gather warps re-pitch each stage unit (8 output rows -> 40 input
    # rows) into a ring of 3 slots per CTA in the workspace, sized for 160 CTAs, whatever the batch
    monkeypatch.setenv("WF_RING", "1")
    d = wf.plan_fold([512, 227, 227, 3], [11, 11, 3, 96], 4, 4, 0, 0, dtype="bf16")["device"]
    assert d["producer"] == "ring+tma" and d["workspace_bytes"] == 160 * 3 * 40 * 232 * 3 * 2
    monkeypatch.delenv("WF_RING")
    # WF_GATHER=1: rows staged in shared memory and realigned by gather warps, no workspace
    monkeypatch.setenv("WF_GATHER", "1")
    d = wf.plan_fold([512, 227, 227, 3], [11, 11, 3, 96], 4, 4, 0, 0, dtype="bf16")["device"]
    assert d["producer"] == "gather" and d["workspace_bytes"] == 0 and d["pitched_w"] == 0
    ref = wf.check_legality([512, 227, 227, 3], [11, 11, 3, 96], 8, stride_h=4, stride_w=4)
    assert ref["status"] == "fallback"  # the reference rule is unchanged


def test_unfolded_variant_plan():
    c = _core.FoldedConv([8, 224, 224, 3], [7, 7, 3, 64], 2, 2, 3, 3, "bf16", 0, 0, "unfolded")
    d = c.device
    assert d["variant"] == "unfolded" and d["producer"] == "im2col" and d["f"] == 1
    assert d["mma_entries"] == 7 * 2  # 21-element window rows in two 16-element K-steps per kh
    assert d["useful_macs"] == 8 * 112 * 112 * 64 * 7 * 7 * 3
    assert c.output_shape == [8, 112, 112, 64]
    with pytest.raises(ValueError):
        _core.FoldedConv([8, 224, 224, 3], [7, 7, 3, 64], 2, 2, 3, 3, "bf16", 0, 0, "sideways")


def test_generalized_legality_reasons():
    # unaligned rows: the re-pitch pass + TMA by default
    assert wf.plan_fold([1, 32, 30, 3], [3, 3, 3, 16], factor=16)["device"]["producer"] == "repitch+tma"
    assert wf.plan_fold([1, 32, 30, 3], [3, 3, 3, 16], factor=4, dtype="tf32")["device"]["producer"] == "repitch+tma"
    assert wf.plan_fold([1, 32, 30, 3], [3, 3, 3, 16], factor=4, dtype="tf32")["device"]["pitched_w"] == 32
    assert wf.plan_fold([1, 32, 32, 3], [3, 3, 3, 16], 2, 3, factor=16)["reason"] == "StrideOnFoldAxis"
    assert wf.plan_fold([1, 32, 32, 3], [3, 3, 3, 16], factor=4)["reason"] == "UnalignedPixel"
    with pytest.raises(wf.ShapeMismatchError):
        wf.plan_fold([1, 32, 32, 3], [3, 3, 4, 16])


def test_folded_filter_shape():
    assert _core.folded_filter_shape([7, 7, 3, 64], 16, 2, 3) == [7, 3, 48, 512]
    assert _core.folded_filter_shape([5, 1, 1, 1], 8) == [5, 1, 8, 8]
    with pytest.raises(wf.IllegalFoldError):
        _core.folded_filter_shape([7, 7, 3, 64], 3, 2, 3)


def test_auto_schedule_choices_for_the_bench_workloads(monkeypatch):
    """Guard the planner's automatic choices (DESIGN 4): cross-kh core-column
    pairs, two M tiles per A stage, no CTA pairs for the headline R50 b8192;
    R50 issued/useful MACs at 1/0.63."""
    for k in ("WF_KPAIR", "WF_TPS", "WF_CTA_PAIR"):
        monkeypatch.delenv(k, raising=False)
    from paper_2601_11608_b200 import _abi as A
    p = A.plan_fold(A.make_desc(8192, 224, 224, 3, 7, 7, 64, 2, 2, 3, 3), 0, 0, A.WF_BF16).as_dict()
    assert (p["kstep_mode"], p["stage_tiles"], p["cta_pair"], p["n_tiles"]) == (1, 2, 1, 1)
    assert p["mma_entries"] == 21
    assert abs(p["useful_macs"] / p["issued_macs"] - 0.631) < 0.005
    # AlexNet zero-padded to Cin 8: B does not fit one SM -> CTA pairs
    p = A.plan_fold(A.make_desc(512, 227, 227, 8, 11, 11, 96, 4, 4, 0, 0), 0, 0, A.WF_BF16).as_dict()
    assert p["status"] == "apply" and p["cta_pair"] == 2
    # batch 1: one output group per N-tile (more CTAs for a latency-bound launch)
    p = A.plan_fold(A.make_desc(1, 224, 224, 3, 7, 7, 64, 2, 2, 3, 3), 0, 0, A.WF_TF32).as_dict()
    assert p["n_tiles"] == 2 and p["stage_tiles"] == 1


def test_wide_pixel_covers_keep_the_no_swizzle_layout():
    """Stride 3 forces f = 24 (9 core columns per folded pixel); a 32-byte-cover schedule would need more
    SWIZZLE_32B regions than a launch holds (4), so the planner keeps the no-swizzle layout (found by
    tests/test_gpu_fuzz.py: the launch used to fail with 'too many SWIZZLE_32B regions')."""
    from paper_2601_11608_b200 import _abi as A
    d = A.schedule_describe(A.make_desc(2, 33, 24, 3, 1, 1, 64, 3, 3, 0, 0), 0, 0, A.WF_BF16)
    assert d["f"] == 24 and d["Q"] == 9 and d["sw32"] == 0
