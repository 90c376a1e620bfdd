"""CPU: the C-ABI shared library loads and exports exactly what
include/widthfold_b200.h declares; host-only entry points behave (no GPU)."""
import ctypes
import os
import re

import pytest

from paper_2601_11608_b200 import _abi as A
from tests.conftest import ROOT

HEADER = os.path.join(ROOT, "include", "widthfold_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(wf_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 12
    lib = A.lib()
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in widthfold_b200.h but not exported"
    assert set(A.EXPORTED) <= set(syms)


def test_abi_version_and_error_channel():
    assert A.lib().wf_abi_version() == 6
    d = A.make_desc(1, 8, 8, 3, 3, 3, 4, 1, 1, 0, 0)
    p = A.FoldPlan()
    # bad dtype -> WF_INVALID_ARGUMENT with a message
    st = A.lib().wf_plan_fold(ctypes.byref(d), 0, 0, A.WF_F32, ctypes.byref(p))
    assert st == A.WF_INVALID_ARGUMENT
    assert b"dtype" in A.lib().wf_last_error()
    bad = A.make_desc(1, 2, 8, 3, 5, 3, 4)
    assert A.lib().wf_plan_fold(ctypes.byref(bad), 0, 0, A.WF_BF16, ctypes.byref(p)) == A.WF_DEGENERATE_OUTPUT
    neg = A.make_desc(1, 8, 8, 0, 3, 3, 4)
    assert A.lib().wf_plan_fold(ctypes.byref(neg), 0, 0, A.WF_BF16, ctypes.byref(p)) == A.WF_SHAPE_MISMATCH


def test_plan_is_deterministic_and_packed_size_positive():
    d = A.make_desc(8192, 224, 224, 3, 7, 7, 64, 2, 2, 3, 3)
    p1 = A.plan_fold(d, 0, 0, A.WF_BF16)
    p2 = A.plan_fold(d, 0, 0, A.WF_BF16)
    assert bytes(p1) == bytes(p2)
    assert p1.status == A.WF_FOLD_APPLY and p1.f == 8 and p1.r == 4
    assert A.lib().wf_packed_filter_bytes(p1) == p1.packed_bytes > 0
    assert p1.table_bytes % 128 == 0


def test_device_calls_fail_cleanly_without_pointers():
    d = A.make_desc(1, 32, 32, 3, 3, 3, 16, 1, 1, 1, 1)
    p = A.plan_fold(d, 16, 0, A.WF_BF16)
    assert A.lib().wf_conv_fold_fwd(None, None, None, None, ctypes.byref(d), ctypes.byref(p), A.WF_BF16, 0,
                                    None) == A.WF_INVALID_ARGUMENT
    assert A.lib().wf_conv_fold_fwd(1, 1, None, 1, ctypes.byref(d), ctypes.byref(p), A.WF_BF16, 0x80,
                                    None) == A.WF_INVALID_ARGUMENT


def test_sms_override_roundtrip():
    A.lib().wf_set_num_sms(74)
    A.lib().wf_set_num_sms(0)
