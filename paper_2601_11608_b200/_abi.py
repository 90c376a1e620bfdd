"""ctypes binding of the C-ABI in include/widthfold_b200.h.

This is the product's own boundary (libwidthfold_b200.so, built in-tree by
``csrc/Makefile``). It fails loudly when the library is missing: there is no
CPU fallback anywhere on the conv path.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, byref, c_char_p, c_int, c_int32, c_int64, c_size_t, c_uint32, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libwidthfold_b200.so")

# wf_status
WF_OK, WF_SHAPE_MISMATCH, WF_DEGENERATE_OUTPUT, WF_ILLEGAL_FOLD = 0, 1, 2, 3
WF_NOT_BLOCK_DIAGONAL, WF_INVALID_ARGUMENT, WF_UNSUPPORTED, WF_CUDA_ERROR = 4, 5, 6, 7
# wf_dtype
WF_F32, WF_TF32, WF_BF16, WF_F16 = 0, 1, 2, 3
# wf_fold_status
WF_FOLD_APPLY, WF_FOLD_FALLBACK = 0, 1
# wf_epilogue
WF_EPI_NONE, WF_EPI_BIAS, WF_EPI_RELU = 0, 1, 2
WF_EPI_PREPITCHED = 4  # the workspace already holds x re-pitched (wf_repitch_input)
WF_EPI_ROW_PRODUCER = 0x4000  # cross-check: the row-gather producer builds the TMA A layout

# FoldReason strings, same order as include/widthfold/fold.hpp:14-23 and
# src/fold.cpp:8-20, plus the two the generalized device fold adds.
REASONS = [
    "None", "WidthNotDivisible", "KernelSpansFoldAxis", "StrideOnFoldAxis", "AlreadyAligned",
    "FactorTooLarge", "UnsupportedChannels", "NotProfitable", "UnalignedPixel", "OutputTail",
]

EXPORTED = [
    "wf_plan_fold", "wf_plan_unfolded", "wf_packed_filter_bytes", "wf_expand_filter_pack", "wf_expand_filter_dense",
    "wf_conv_fold_fwd", "wf_conv_fold_fwd_ws", "wf_set_num_sms", "wf_last_error", "wf_abi_version",
    "wf_schedule_describe", "wf_cast_f32", "wf_conv_grouped_fwd", "wf_repitch_input",
]


class ConvDesc(ctypes.Structure):
    _fields_ = [(n, c_int64) for n in
                ("n", "h", "w", "c", "kh", "kw", "cout", "stride_h", "stride_w", "pad_h", "pad_w")]


class FoldPlan(ctypes.Structure):
    _fields_ = [
        ("status", c_int32), ("reason", c_int32),
        ("f", c_int64), ("r", c_int64), ("c0", c_int64), ("kw_f", c_int64), ("k_f", c_int64),
        ("cout_f", c_int64),
        ("in_dtype", c_int32), ("elem_bytes", c_int32),
        ("oh", c_int64), ("ow", c_int64), ("wf", c_int64), ("wfo", c_int64),
        ("units_per_px", c_int64), ("group_size", c_int64), ("n_groups", c_int64),
        ("n_tiles", c_int64), ("tile_rows", c_int64), ("wbox", c_int64), ("nrows", c_int64),
        ("mma_entries", c_int64), ("table_bytes", c_int64), ("packed_bytes", c_int64), ("epi_chunk", c_int64), ("variant", c_int32), ("producer", c_int32), ("cta_pair", c_int32),
        ("stage_tiles", c_int32), ("kstep_mode", c_int32), ("launch_opts", c_int32),
        ("pitched_w", c_int64), ("workspace_bytes", c_int64),
        ("useful_macs", c_uint64), ("issued_macs", c_uint64),
    ]

    def as_dict(self) -> dict:
        d = {name: getattr(self, name) for name, _ in self._fields_}
        d["status"] = "apply" if self.status == WF_FOLD_APPLY else "fallback"
        d["reason"] = REASONS[self.reason] if 0 <= self.reason < len(REASONS) else "?"
        return d


class WidthfoldError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


_lib = None


def lib() -> ctypes.CDLL:
    """Load libwidthfold_b200.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: run `make -C paper_2601_11608_b200/csrc` "
                "(or __graft_entry__.build()). There is no CPU fallback.")
        L = ctypes.CDLL(LIB_PATH)
        L.wf_plan_fold.argtypes = [POINTER(ConvDesc), c_int64, c_int64, c_int, POINTER(FoldPlan)]
        L.wf_plan_fold.restype = c_int
        L.wf_plan_unfolded.argtypes = [POINTER(ConvDesc), c_int, POINTER(FoldPlan)]
        L.wf_plan_unfolded.restype = c_int
        L.wf_packed_filter_bytes.argtypes = [POINTER(FoldPlan)]
        L.wf_packed_filter_bytes.restype = c_size_t
        L.wf_expand_filter_pack.argtypes = [c_void_p, c_void_p, POINTER(ConvDesc), POINTER(FoldPlan),
                                            c_void_p, c_void_p, c_void_p]
        L.wf_expand_filter_pack.restype = c_int
        L.wf_expand_filter_dense.argtypes = [c_void_p, POINTER(ConvDesc), c_int64, c_void_p, c_void_p]
        L.wf_expand_filter_dense.restype = c_int
        L.wf_conv_fold_fwd.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, POINTER(ConvDesc),
                                       POINTER(FoldPlan), c_int, c_uint32, c_void_p]
        L.wf_conv_fold_fwd.restype = c_int
        L.wf_conv_fold_fwd_ws.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, POINTER(ConvDesc),
                                          POINTER(FoldPlan), c_int, c_uint32, c_void_p]
        L.wf_conv_fold_fwd_ws.restype = c_int
        L.wf_repitch_input.argtypes = [c_void_p, c_void_p, POINTER(ConvDesc), POINTER(FoldPlan), c_void_p]
        L.wf_repitch_input.restype = c_int
        L.wf_set_num_sms.argtypes = [c_int]
        L.wf_set_num_sms.restype = None
        L.wf_last_error.argtypes = []
        L.wf_last_error.restype = c_char_p
        L.wf_abi_version.argtypes = []
        L.wf_abi_version.restype = c_int
        L.wf_schedule_describe.argtypes = [POINTER(ConvDesc), c_int64, c_int64, c_int, ctypes.c_char_p, c_size_t]
        L.wf_schedule_describe.restype = c_int
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != WF_OK:
        msg = lib().wf_last_error().decode(errors="replace")
        raise WidthfoldError(status, msg or f"widthfold status {status}")


def make_desc(n, h, w, c, kh, kw, cout, stride_h=1, stride_w=1, pad_h=0, pad_w=0) -> ConvDesc:
    return ConvDesc(n, h, w, c, kh, kw, cout, stride_h, stride_w, pad_h, pad_w)


def plan_unfolded(desc: ConvDesc, in_dtype: int = WF_BF16) -> FoldPlan:
    p = FoldPlan()
    check(lib().wf_plan_unfolded(byref(desc), in_dtype, byref(p)))
    return p


def plan_fold(desc: ConvDesc, f: int = 0, group_size: int = 0, in_dtype: int = WF_BF16) -> FoldPlan:
    p = FoldPlan()
    check(lib().wf_plan_fold(byref(desc), f, group_size, in_dtype, byref(p)))
    return p


def schedule_describe(desc: ConvDesc, f: int = 0, group_size: int = 0, in_dtype: int = WF_BF16) -> dict:
    """The tcgen05 schedule of a plan (diagnostic; tests replay it on the CPU)."""
    import json
    buf = ctypes.create_string_buffer(1 << 20)
    check(lib().wf_schedule_describe(byref(desc), f, group_size, in_dtype, buf, len(buf)))
    return json.loads(buf.value.decode())
