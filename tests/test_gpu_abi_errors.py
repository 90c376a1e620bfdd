"""The C-ABI rejects bad calls with a status and a message instead of faulting (driven through ctypes,
the way a reference-side binding would call it)."""
import ctypes

import pytest
import torch

from paper_2601_11608_b200 import _abi as A

pytestmark = pytest.mark.gpu


def _setup(n=2, h=64, w=64, k=7, co=64, s=2, p=3):
    d = A.make_desc(n, h, w, 3, k, k, co, s, s, p, p)
    plan = A.plan_fold(d, 0, 0, A.WF_BF16)
    L = A.lib()
    packed = torch.empty(L.wf_packed_filter_bytes(ctypes.byref(plan)), dtype=torch.uint8, device="cuda")
    wt = (torch.randn(k, k, 3, co, device="cuda") * 0.1).bfloat16()
    b = torch.randn(co, device="cuda")
    brep = torch.empty(plan.cout_f, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    A.check(L.wf_expand_filter_pack(wt.data_ptr(), b.data_ptr(), ctypes.byref(d), ctypes.byref(plan),
                                    packed.data_ptr(), brep.data_ptr(), st))
    oh = (h + 2 * p - k) // s + 1
    x = torch.zeros(n * h * w * 3 + 64, dtype=torch.bfloat16, device="cuda")
    y = torch.zeros(n * oh * oh * co + 64, dtype=torch.bfloat16, device="cuda")
    return L, d, plan, packed, brep, x, y, st


def _fwd(L, d, plan, packed, brep, xp, yp, st, epi=A.WF_EPI_BIAS, ws=None):
    return L.wf_conv_fold_fwd_ws(xp, ws, packed.data_ptr(), brep.data_ptr(), yp, ctypes.byref(d),
                                 ctypes.byref(plan), A.WF_BF16, epi, st)


def test_good_call_then_rejections():
    L, d, plan, packed, brep, x, y, st = _setup()
    assert _fwd(L, d, plan, packed, brep, x.data_ptr(), y.data_ptr(), st) == A.WF_OK
    torch.cuda.synchronize()
    # x not 16-byte aligned, y not 32-byte aligned
    assert _fwd(L, d, plan, packed, brep, x.data_ptr() + 2, y.data_ptr(), st) == A.WF_INVALID_ARGUMENT
    assert b"aligned" in L.wf_last_error()
    assert _fwd(L, d, plan, packed, brep, x.data_ptr(), y.data_ptr() + 16, st) == A.WF_INVALID_ARGUMENT
    # unknown epilogue bits (the profiling switches are rejected by a release build)
    assert _fwd(L, d, plan, packed, brep, x.data_ptr(), y.data_ptr(), st, epi=0x100) == A.WF_INVALID_ARGUMENT
    # null pointers
    assert L.wf_conv_fold_fwd_ws(None, None, packed.data_ptr(), None, y.data_ptr(), ctypes.byref(d),
                                 ctypes.byref(plan), A.WF_BF16, 0, st) == A.WF_INVALID_ARGUMENT
    # a plan built for another descriptor
    d2 = A.make_desc(2, 64, 64, 3, 3, 3, 64, 1, 1, 1, 1)
    assert L.wf_conv_fold_fwd_ws(x.data_ptr(), None, packed.data_ptr(), brep.data_ptr(), y.data_ptr(),
                                 ctypes.byref(d2), ctypes.byref(plan), A.WF_BF16, A.WF_EPI_BIAS, st) != A.WF_OK
    torch.cuda.synchronize()  # the stream is still healthy
    assert _fwd(L, d, plan, packed, brep, x.data_ptr(), y.data_ptr(), st) == A.WF_OK
    torch.cuda.synchronize()


def test_workspace_required_for_unaligned_rows():
    L, d, plan, packed, brep, x, y, st = _setup(n=2, h=67, w=67, k=11, co=96, s=4, p=0)
    assert plan.workspace_bytes > 0
    assert _fwd(L, d, plan, packed, brep, x.data_ptr(), y.data_ptr(), st) == A.WF_INVALID_ARGUMENT
    assert b"workspace" in L.wf_last_error()
    ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device="cuda")
    assert L.wf_repitch_input(x.data_ptr(), None, ctypes.byref(d), ctypes.byref(plan), st) == A.WF_INVALID_ARGUMENT
    assert L.wf_repitch_input(x.data_ptr(), ws.data_ptr(), ctypes.byref(d), ctypes.byref(plan), st) == A.WF_OK
    assert _fwd(L, d, plan, packed, brep, x.data_ptr(), y.data_ptr(), st, epi=A.WF_EPI_BIAS | A.WF_EPI_PREPITCHED,
                ws=ws.data_ptr()) == A.WF_OK
    torch.cuda.synchronize()
