"""Device-side fold ops over CUDA torch tensors, calling the C-ABI.

torch is plumbing here (device memory + streams); the arithmetic is the
sm_100a kernels in libwidthfold_b200.so. Nothing in this module falls back to
a CPU or library implementation: a missing library or a non-CUDA tensor is an
error.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import _abi as A

_TORCH_TO_WF = {torch.bfloat16: A.WF_BF16, torch.float16: A.WF_F16, torch.float32: A.WF_TF32}
_OUT_TO_WF = {torch.bfloat16: A.WF_BF16, torch.float16: A.WF_F16, torch.float32: A.WF_F32}


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _require_cuda(*ts: torch.Tensor) -> None:
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("widthfold_b200 device ops need CUDA tensors (no CPU fallback)")


@dataclass
class FoldedFilter:
    """The once-per-weights state: plan + packed tcgen05 B operand + replicated bias.

    Mirrors the reference's FoldResult filter/bias halves (include/widthfold/fold.hpp:81-86),
    but the filter lives in the MMA operand layout instead of a dense tensor.
    """

    desc: A.ConvDesc
    plan: A.FoldPlan
    packed: torch.Tensor
    bias_rep: torch.Tensor | None
    in_dtype: torch.dtype
    extra: dict = field(default_factory=dict)

    @property
    def plan_dict(self) -> dict:
        return self.plan.as_dict()


def make_desc_for(x_shape, w_shape, stride=(1, 1), padding=(0, 0)) -> A.ConvDesc:
    n, h, w, c = x_shape
    kh, kw, c2, cout = w_shape
    if c2 != c:
        raise ValueError(f"filter Cin {c2} != input Cin {c}")
    return A.make_desc(n, h, w, c, kh, kw, cout, stride[0], stride[1], padding[0], padding[1])


def prepare_filter(w: torch.Tensor, b: torch.Tensor | None, x_shape, stride=(1, 1), padding=(0, 0),
                   fold: int = 0, group_size: int = 0) -> FoldedFilter:
    """Plan the fold for (x_shape, w) and expand+pack w (and replicate b) on device."""
    _require_cuda(w, b)
    in_dtype = w.dtype
    if in_dtype not in _TORCH_TO_WF:
        raise ValueError(f"unsupported filter dtype {in_dtype}")
    desc = make_desc_for(tuple(x_shape), tuple(w.shape), stride, padding)
    plan = A.plan_fold(desc, fold, group_size, _TORCH_TO_WF[in_dtype])
    if plan.status != A.WF_FOLD_APPLY:
        raise A.WidthfoldError(A.WF_UNSUPPORTED,
                               f"fold not applicable: {A.REASONS[plan.reason]} (f={plan.f})")
    packed = torch.empty(A.lib().wf_packed_filter_bytes(plan), dtype=torch.uint8, device=w.device)
    bias_rep = None
    if b is not None:
        b = b.to(device=w.device, dtype=torch.float32).contiguous()
        bias_rep = torch.empty(plan.cout_f, dtype=torch.float32, device=w.device)
    w = w.contiguous()
    A.check(A.lib().wf_expand_filter_pack(_ptr(w), _ptr(b), desc, plan, _ptr(packed), _ptr(bias_rep),
                                          _stream_ptr(w.device)))
    return FoldedFilter(desc, plan, packed, bias_rep, in_dtype, {"w": w})


def conv_folded(x: torch.Tensor, ff: FoldedFilter, *, relu: bool = False, bias: bool = True,
                out: torch.Tensor | None = None, out_dtype: torch.dtype | None = None,
                _profile_flags: int = 0) -> torch.Tensor:
    """y = ReLU?(conv(x, w) + b) through the folded tcgen05 kernel (NHWC in, NHWC out).

    ``_profile_flags`` (0x100 skip MMAs, 0x200 skip epilogue, 0x400 skip stores) exist
    only to decompose the kernel's time in profiling runs; results are garbage with them.
    """
    _require_cuda(x)
    if x.dtype != ff.in_dtype:
        raise ValueError(f"x dtype {x.dtype} != packed filter dtype {ff.in_dtype}")
    d = ff.desc
    if tuple(x.shape) != (d.n, d.h, d.w, d.c):
        raise ValueError(f"x shape {tuple(x.shape)} != planned {(d.n, d.h, d.w, d.c)}")
    x = x.contiguous()
    out_dtype = out_dtype or (torch.float32 if x.dtype == torch.float32 else x.dtype)
    shape = (d.n, ff.plan.oh, ff.plan.ow, d.cout)
    if out is None:
        out = torch.empty(shape, dtype=out_dtype, device=x.device)
    elif tuple(out.shape) != shape or out.dtype != out_dtype or not out.is_contiguous():
        raise ValueError("bad output buffer")
    epi = 0
    if bias and ff.bias_rep is not None:
        epi |= A.WF_EPI_BIAS
    if relu:
        epi |= A.WF_EPI_RELU
    epi |= _profile_flags & 0x700
    A.check(A.lib().wf_conv_fold_fwd(_ptr(x), _ptr(ff.packed), _ptr(ff.bias_rep) if epi & A.WF_EPI_BIAS else None,
                                     _ptr(out), d, ff.plan, _OUT_TO_WF[out_dtype], epi, _stream_ptr(x.device)))
    return out


def expand_filter_dense(w: torch.Tensor, f: int, stride_w: int = 1, pad_w: int = 0) -> torch.Tensor:
    """Dense generalized expansion W'(KH, KW', f*C, r*Cout) of an fp32 filter, on device."""
    _require_cuda(w)
    if w.dtype != torch.float32:
        raise ValueError("expand_filter_dense takes an fp32 filter (bit-exact transform)")
    kh, kw, c, cout = w.shape
    desc = A.make_desc(1, kh, kw + f, c, kh, kw, cout, 1, stride_w, 0, pad_w)
    r = f // stride_w
    c0 = -((pad_w + f - 1) // f)
    kwf = (f - stride_w - pad_w + kw - 1) // f - c0 + 1
    out = torch.empty((kh, kwf, f * c, r * cout), dtype=torch.float32, device=w.device)
    A.check(A.lib().wf_expand_filter_dense(_ptr(w.contiguous()), desc, f, _ptr(out), _stream_ptr(w.device)))
    return out
