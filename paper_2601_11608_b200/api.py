"""Reference-compatible Python API (the drop-in for ``widthfold``).

Every name of the reference package (/root/reference/proj/python/widthfold/
__init__.py:5-49) is provided with the same positional/keyword arguments,
return conventions and exception types (ShapeMismatchError, IllegalFoldError,
DegenerateOutputError are ``ValueError`` subclasses, bindings.cpp:51-56).
Additions are keyword-only (``padding``, ``bias``, ``relu``, ``precision``...).

Arrays: numpy inputs behave like the reference (copied in, result returned as
numpy float32); CUDA torch tensors are used in place and results stay on the
device. All arithmetic runs in this package's sm_100a kernels through the
C++ host layer (``_core``) and the C-ABI; there is no CPU compute path.

Precision: fp32 inputs default to ``precision="exact"`` -- the CUDA-core
kernel that reproduces the reference conv2d bit-for-bit (kh -> kw -> ci
order, no FMA). ``precision="tf32"``, or bf16/fp16 inputs, run the folded
tcgen05 tensor-core kernel (within 1e-3 / 1e-2 normwise of the fp32 result).
"""
from __future__ import annotations

import weakref
from typing import Any

import numpy as np
import torch

from . import _core

ShapeMismatchError = _core.ShapeMismatchError
IllegalFoldError = _core.IllegalFoldError
DegenerateOutputError = _core.DegenerateOutputError
NotBlockDiagonalError = _core.NotBlockDiagonalError
UnsupportedError = _core.UnsupportedError

check_legality = _core.check_legality
choose_fold_factor = _core.choose_fold_factor
count_macs = _core.count_macs
mac_report = _core.mac_report
plan_fold = _core.plan_fold

_DT_NAME = {torch.bfloat16: "bf16", torch.float16: "f16", torch.float32: "tf32"}
_OUT_NAME = {torch.bfloat16: "bf16", torch.float16: "f16", torch.float32: "f32"}
_PREC_DTYPE = {"bf16": torch.bfloat16, "fp16": torch.float16, "f16": torch.float16, "tf32": torch.float32}


# ----------------------------------------------------------------- plumbing
def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("widthfold_b200 needs a CUDA device (sm_100a); there is no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


def _stream(dev: torch.device) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


# the current stream's raw cudaStream_t without building a torch.cuda.Stream
# object (the per-call path of FoldedConv2d; several us cheaper)
_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _as_tensor(a, dtype=None) -> tuple[torch.Tensor, bool]:
    """(device tensor, came_from_numpy)."""
    if isinstance(a, torch.Tensor):
        if not a.is_cuda:
            t = a.to(_device())
            return (t if dtype is None else t.to(dtype)).contiguous(), True
        return (a if dtype is None else a.to(dtype)).contiguous(), False
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    t = torch.from_numpy(arr).to(_device(), non_blocking=False)
    return (t if dtype is None else t.to(dtype)).contiguous(), True


def _ret(t: torch.Tensor, host: bool):
    if host:
        return t.float().cpu().numpy()
    return t


def _ptr(t: torch.Tensor | None) -> int:
    return 0 if t is None else t.data_ptr()


def _pair(v) -> tuple[int, int]:
    if isinstance(v, (tuple, list)):
        return int(v[0]), int(v[1])
    return int(v), int(v)


# ------------------------------------------------------ folded tensor-core conv
class FoldedConv2d:
    """Once-per-weights folded convolution (the product hot path).

    Plans the generalized width fold for ``input_shape``, expands and packs the
    filter into the tcgen05 operand layout on the device, replicates the bias,
    then runs ``y = ReLU?(conv(x, w) + b)`` per call with NHWC in and out.
    """

    def __init__(self, w: torch.Tensor, b: torch.Tensor | None, input_shape, stride=1, padding=0,
                 dtype: torch.dtype | None = None, fold: int = 0, group_size: int = 0, variant: str = "fold"):
        w, _ = _as_tensor(w)
        dtype = dtype or w.dtype
        if dtype not in _DT_NAME:
            raise ValueError(f"unsupported compute dtype {dtype}")
        w = w.to(dtype).contiguous()
        sh, sw = _pair(stride)
        ph, pw = _pair(padding)
        self.input_shape = tuple(int(v) for v in input_shape)
        self.dtype = dtype
        self.variant = variant
        self.core = _core.FoldedConv(list(self.input_shape), list(w.shape), sh, sw, ph, pw,
                                     _DT_NAME[dtype], fold, group_size, variant)
        dev = w.device
        self.packed = torch.empty(self.core.packed_bytes, dtype=torch.uint8, device=dev)
        self.b_rep = None
        bf = None
        if b is not None:
            bf, _ = _as_tensor(b, torch.float32)
            self.b_rep = torch.empty(self.core.cout_f, dtype=torch.float32, device=dev)
        self.core.pack(w.data_ptr(), _ptr(bf), self.packed.data_ptr(), _ptr(self.b_rep), _stream(dev))
        self._keep = (w, bf)
        # re-pitched input (rows whose pitch is not TMA-addressable, e.g. AlexNet W=227)
        self.workspace = (torch.empty(self.core.workspace_bytes, dtype=torch.uint8, device=dev)
                          if self.core.workspace_bytes else None)
        self._geom = (sh, sw, ph, pw)
        self.output_shape = tuple(self.core.output_shape)
        self._out_default = torch.float32 if self.dtype == torch.float32 else self.dtype
        self._set_ptrs()

    def _set_ptrs(self) -> None:
        """Device pointers the per-call path passes (re-taken whenever a buffer is replaced)."""
        self._packed_ptr = self.packed.data_ptr()
        self._brep_ptr = _ptr(self.b_rep)
        self._ws_ptr = _ptr(self.workspace)

    @property
    def plan(self) -> dict:
        return self.core.plan

    @property
    def device_plan(self) -> dict:
        return self.core.device

    def __call__(self, x: torch.Tensor, *, relu: bool = False, bias: bool = True, out: torch.Tensor | None = None,
                 out_dtype: torch.dtype | None = None) -> torch.Tensor:
        """y = ReLU?(conv(x, w) + b) into ``out`` (allocated when None), stream-ordered."""
        return self._forward(x, relu, bias, out, out_dtype, 0)

    def _forward(self, x: torch.Tensor, relu: bool = False, bias: bool = True, out: torch.Tensor | None = None,
                 out_dtype: torch.dtype | None = None, flags: int = 0) -> torch.Tensor:
        """__call__ with extra wf_conv_fold_fwd epilogue bits: tests and tools
        only (``_abi.WF_EPI_ROW_PRODUCER`` cross-check; the 0xFFFF00 profiling
        switches need a ``make PROFILE=1`` build and are rejected otherwise).

        The per-call path is kept lean (batch-1 latency is host-bound): cheap
        checks, the raw current stream, and pointers precomputed at plan time;
        the C++ side reuses the launch prepared for these buffers."""
        if not (isinstance(x, torch.Tensor) and x.is_cuda):
            raise ValueError("FoldedConv2d takes a CUDA tensor (use conv2d() for numpy inputs)")
        if x.dtype != self.dtype:
            raise ValueError(f"x dtype {x.dtype} != planned {self.dtype}")
        if x.shape != self.input_shape:
            raise ShapeMismatchError(f"x shape {tuple(x.shape)} != planned {self.input_shape}")
        if not x.is_contiguous():
            x = x.contiguous()
        if out_dtype is None:
            out_dtype = self._out_default
        if out is None:
            out = torch.empty(self.output_shape, dtype=out_dtype, device=x.device)
        elif out.shape != self.output_shape or out.dtype != out_dtype or not out.is_contiguous():
            raise ShapeMismatchError("output buffer has the wrong shape/dtype/layout")
        use_bias = bias and self._brep_ptr != 0
        dev = x.get_device()
        stream = _raw_stream(dev) if _raw_stream is not None else _stream(x.device)
        self.core.forward(x.data_ptr(), self._packed_ptr, self._brep_ptr if use_bias else 0, out.data_ptr(),
                          _OUT_NAME[out_dtype], use_bias, relu, stream, flags, self._ws_ptr)
        return out


    def graphed(self, x: torch.Tensor, out: torch.Tensor | None = None, *, relu: bool = False, bias: bool = True):
        """Capture one forward on the static buffers ``x`` / ``out`` into a CUDA
        graph; returns ``(replay, out)``. ``replay()`` re-runs the conv on
        whatever ``x`` holds, without host launch overhead (R50 b1 TF32: ~5.3 us
        per replayed launch vs ~5.8 us eager back to back and ~5 us of host
        time per eager call, tools/host_path_probe.py)."""
        if out is None:
            out_dtype = torch.float32 if self.dtype == torch.float32 else self.dtype
            out = torch.empty(self.output_shape, dtype=out_dtype, device=x.device)
        self(x, relu=relu, bias=bias, out=out)  # plans/caches the schedule outside the capture
        side = torch.cuda.Stream(x.device)
        side.wait_stream(torch.cuda.current_stream(x.device))
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(side):
            with torch.cuda.graph(graph, stream=side):
                self(x, relu=relu, bias=bias, out=out)
        torch.cuda.current_stream(x.device).wait_stream(side)
        return graph.replay, out

    # plan fields that scale with the batch but leave the packed operand (the
    # schedule table + B layout) unchanged; every other field must match to share it
    _BATCH_COUNTERS = ("useful_macs", "issued_macs", "workspace_bytes")

    def with_batch(self, n: int) -> "FoldedConv2d":
        """Same filter for batch ``n``, with its own workspace. The packed operand
        is shared when the batch-``n`` plan has the same schedule (N-tiling,
        stage tiles, CTA pairs, K-step mode...); otherwise the filter is packed
        again for the new plan (a batch-dependent planner choice never runs
        against a mismatched operand)."""
        other = object.__new__(FoldedConv2d)
        other.__dict__.update(self.__dict__)
        shape = (int(n),) + self.input_shape[1:]
        sh, sw, ph, pw = self._geom
        w, bf = self._keep
        other.core = _core.FoldedConv(list(shape), list(w.shape), sh, sw, ph, pw, _DT_NAME[self.dtype],
                                      self.core.device["f"] if self.variant == "fold" else 0,
                                      self.core.device["group_size"] if self.variant == "fold" else 0, self.variant)
        mine = {k: v for k, v in self.core.device.items() if k not in self._BATCH_COUNTERS}
        theirs = {k: v for k, v in other.core.device.items() if k not in self._BATCH_COUNTERS}
        dev = self.packed.device
        if mine != theirs:
            other.packed = torch.empty(other.core.packed_bytes, dtype=torch.uint8, device=dev)
            other.b_rep = None if self.b_rep is None else torch.empty_like(self.b_rep)
            other.core.pack(w.data_ptr(), _ptr(bf), other.packed.data_ptr(), _ptr(other.b_rep), _stream(dev))
        other.workspace = (torch.empty(other.core.workspace_bytes, dtype=torch.uint8, device=dev)
                           if other.core.workspace_bytes else None)
        other.input_shape = shape
        other.output_shape = tuple(other.core.output_shape)
        other._set_ptrs()
        return other

    def run_host(self, x_host: torch.Tensor, y_host: torch.Tensor, *, chunk: int = 512, relu: bool = False,
                 bias: bool = True) -> torch.Tensor:
        """End to end from host memory: pinned x_host (N,H,W,C) -> y_host (N,OH,OW,Cout).

        Chunks of ``chunk`` images alternate over two streams, so the H2D copy of
        one chunk, the folded conv of another and the D2H copy of a third overlap.
        Each stream has its own input/output buffers and its own conv (and so
        its own workspace for plans that re-pitch the input), so concurrent
        chunks never share scratch memory.
        """
        if x_host.is_cuda or y_host.is_cuda:
            raise ValueError("run_host takes host tensors (pinned for overlap)")
        n = x_host.shape[0]
        dev = self.packed.device
        chunk = max(1, min(chunk, n))
        convs = {}
        streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
        cur = torch.cuda.current_stream(dev)
        for s in streams:
            s.wait_stream(cur)
        xbufs = [torch.empty((chunk,) + self.input_shape[1:], dtype=self.dtype, device=dev) for _ in range(2)]
        ybufs = [torch.empty((chunk,) + self.output_shape[1:], dtype=y_host.dtype, device=dev) for _ in range(2)]
        for i, start in enumerate(range(0, n, chunk)):
            m = min(chunk, n - start)
            k = i & 1
            with torch.cuda.stream(streams[k]):
                conv = convs.get((m, k))
                if conv is None:
                    conv = convs[(m, k)] = self.with_batch(m)
                xd, yd = xbufs[k][:m], ybufs[k][:m]
                xd.copy_(x_host[start:start + m], non_blocking=True)
                conv(xd, relu=relu, bias=bias, out=yd, out_dtype=y_host.dtype)
                y_host[start:start + m].copy_(yd, non_blocking=True)
        for s in streams:
            cur.wait_stream(s)
        return y_host


_FOLD_CACHE: dict[Any, tuple[Any, FoldedConv2d]] = {}


def _cached_folded(w: torch.Tensor, b: torch.Tensor | None, xshape, stride, padding, dtype, fold, group_size):
    key = (w.data_ptr(), w._version, tuple(w.shape), None if b is None else (b.data_ptr(), b._version),
           tuple(xshape), stride, padding, dtype, fold, group_size)
    hit = _FOLD_CACHE.get(key)
    if hit is not None and hit[0]() is w:
        return hit[1]
    fc = FoldedConv2d(w, b, xshape, stride, padding, dtype, fold, group_size)
    if len(_FOLD_CACHE) > 64:
        _FOLD_CACHE.clear()
    _FOLD_CACHE[key] = (weakref.ref(w), fc)
    return fc


# ----------------------------------------------------------- reference names
def conv2d(x, w, stride_h: int = 1, stride_w: int = 1, *, padding=0, bias=None, relu: bool = False,
           precision: str | None = None, out_dtype: torch.dtype | None = None, fold: int = 0,
           group_size: int = 0):
    """NHWC convolution (reference: widthfold::conv2d, src/refconv.cpp:34-80).

    VALID by default like the reference; ``padding`` adds symmetric zero
    padding. ``bias``/``relu`` fuse the bias_add (+ReLU) epilogue.
    """
    ph, pw = _pair(padding)
    host = not (isinstance(x, torch.Tensor) and x.is_cuda)
    xdt = x.dtype if isinstance(x, torch.Tensor) else torch.float32
    if precision is None:
        precision = "exact" if xdt == torch.float32 else _DT_NAME[xdt]
    if precision == "exact":
        xt, _ = _as_tensor(x, torch.float32)
        wt, _ = _as_tensor(w, torch.float32)
        if xt.dim() != 4 or wt.dim() != 4:
            raise ShapeMismatchError("conv input/filter must be rank-4 (NHWC / HWIO)")
        B, H, W, C = xt.shape
        KH, KW, _, Co = wt.shape
        OH = (H + 2 * ph - KH) // stride_h + 1
        OW = (W + 2 * pw - KW) // stride_w + 1
        y = torch.empty((B, max(OH, 0), max(OW, 0), Co), dtype=torch.float32, device=xt.device)
        _core.conv2d_exact(xt.data_ptr(), wt.data_ptr(), y.data_ptr(), list(xt.shape), list(wt.shape),
                           stride_h, stride_w, ph, pw, _stream(xt.device))
        if bias is not None or relu:
            bt = _as_tensor(bias, torch.float32)[0] if bias is not None else torch.zeros(
                Co, dtype=torch.float32, device=y.device)
            _core.bias_add(y.data_ptr(), bt.data_ptr(), y.data_ptr(), y.numel(), Co, relu, _stream(y.device))
        return _ret(y, host)
    dtype = _PREC_DTYPE[precision]
    xt, _ = _as_tensor(x, dtype)
    wt, _ = _as_tensor(w, dtype)
    bt = None if bias is None else _as_tensor(bias, torch.float32)[0]
    fc = _cached_folded(wt, bt, tuple(xt.shape), (stride_h, stride_w), (ph, pw), dtype, fold, group_size)
    y = fc(xt, relu=relu, bias=bt is not None, out_dtype=out_dtype)
    return _ret(y, host)


def bias_add(y, b, *, relu: bool = False):
    """y'[..., c] = y[..., c] + b[c] (reference: src/refconv.cpp:82-95)."""
    yt, host = _as_tensor(y, torch.float32)
    bt, _ = _as_tensor(b, torch.float32)
    if yt.dim() < 1 or bt.dim() != 1 or bt.shape[0] != yt.shape[-1]:
        raise ShapeMismatchError(f"bias length {tuple(bt.shape)} does not match channel extent of {tuple(yt.shape)}")
    out = torch.empty_like(yt)
    _core.bias_add(yt.data_ptr(), bt.data_ptr(), out.data_ptr(), yt.numel(), bt.shape[0], relu, _stream(yt.device))
    return _ret(out, host)


def conv1d_h(x, w, bias: float = 0.0):
    """Height-only conv of an (H, W, 1) tensor with a (K,) kernel (src/refconv.cpp:97-114)."""
    xt, host = _as_tensor(x, torch.float32)
    wt, _ = _as_tensor(w, torch.float32)
    if xt.dim() != 3 or xt.shape[2] != 1:
        raise ShapeMismatchError(f"conv1d_h input must be (H, W, 1), got {tuple(xt.shape)}")
    if wt.dim() != 1:
        raise ShapeMismatchError(f"conv1d_h kernel must be rank-1, got {tuple(wt.shape)}")
    H, W, _ = xt.shape
    K = wt.shape[0]
    if K > H:
        raise ShapeMismatchError("kernel length exceeds height")
    b = torch.full((1,), float(bias), dtype=torch.float32, device=xt.device)
    y = conv2d(xt.reshape(1, H, W, 1), wt.reshape(K, 1, 1, 1), bias=b)
    return _ret(y.reshape(H - K + 1, W, 1), host)


def _check_factor(factor: int) -> None:
    if factor < 1:
        raise ValueError("fold factor must be >= 1")


def _view_or_copy(t: torch.Tensor, shape, host: bool):
    v = t.reshape(shape)  # row-major identity: a zero-copy view on the device
    return _ret(v, host)


def fold_input(x, factor: int):
    """X'(b,h,w',f) = X(b,h,F*w'+f,0): a reshape (src/fold.cpp:92-111)."""
    _check_factor(factor)
    xt, host = _as_tensor(x)
    if xt.dim() != 4:
        raise IllegalFoldError(f"fold_input wants a rank-4 NHWC tensor, got {tuple(xt.shape)}")
    B, H, W, C = xt.shape
    if C != 1:
        raise IllegalFoldError(f"fold_input requires Cin == 1, got {C}")
    if W % factor:
        raise IllegalFoldError(f"width {W} not divisible by {factor}")
    return _view_or_copy(xt, (B, H, W // factor, factor), host)


def fold_input_general(x, factor: int):
    """X_f[b,h,w',f*C+c] = X[b,h,F*w'+f,c]: a zero-copy NHWC view (src/fold.cpp:113-143)."""
    _check_factor(factor)
    xt, host = _as_tensor(x)
    if xt.dim() != 4:
        raise IllegalFoldError(f"fold_input_general wants a rank-4 NHWC tensor, got {tuple(xt.shape)}")
    B, H, W, C = xt.shape
    if W % factor:
        raise IllegalFoldError(f"width {W} not divisible by {factor}")
    return _view_or_copy(xt, (B, H, W // factor, C * factor), host)


def unfold_input_general(x_f, factor: int):
    """Inverse of fold_input_general (src/fold.cpp:145-175)."""
    _check_factor(factor)
    xt, host = _as_tensor(x_f)
    if xt.dim() != 4:
        raise IllegalFoldError(f"unfold_input_general wants a rank-4 tensor, got {tuple(xt.shape)}")
    B, H, Wf, Cf = xt.shape
    if Cf % factor:
        raise IllegalFoldError(f"channel extent {Cf} not divisible by {factor}")
    return _view_or_copy(xt, (B, H, Wf * factor, Cf // factor), host)


def reconstruct_output(y_folded, factor: int):
    """Inverse index map of the folded output, a reshape (src/fold.cpp:228-259)."""
    _check_factor(factor)
    yt, host = _as_tensor(y_folded)
    if yt.dim() != 4:
        raise ShapeMismatchError(f"reconstruct_output wants a rank-4 tensor, got {tuple(yt.shape)}")
    B, H, Wf, Cf = yt.shape
    if Cf % factor:
        raise ShapeMismatchError(f"channel extent {Cf} not divisible by fold factor {factor}")
    return _view_or_copy(yt, (B, H, Wf * factor, Cf // factor), host)


def expand_filter_general(w, factor: int):
    """Block-diagonal expansion (KH,1,C,Co) -> (KH,1,F*C,F*Co) (src/fold.cpp:185-211), on device."""
    _check_factor(factor)
    wt, host = _as_tensor(w, torch.float32)
    if wt.dim() != 4:
        raise IllegalFoldError(f"expand_filter wants a rank-4 filter, got {tuple(wt.shape)}")
    KH, KW, C, Co = wt.shape
    out = torch.empty((KH, 1, C * factor, Co * factor), dtype=torch.float32, device=wt.device)
    _core.expand_filter_general(wt.data_ptr(), list(wt.shape), factor, out.data_ptr(), _stream(wt.device))
    return _ret(out, host)


def expand_filter(w, factor: int):
    """Diagonal replication of a (KH,1,1,Co) filter (src/fold.cpp:177-183)."""
    wt, host = _as_tensor(w, torch.float32)
    if wt.dim() != 4 or wt.shape[2] != 1:
        raise IllegalFoldError(f"expand_filter wants a (KH, 1, 1, Cout) filter, got {tuple(wt.shape)}")
    return _ret(expand_filter_general(wt, factor), host)


def expand_filter_folded(w, factor: int, stride_w: int = 1, pad_w: int = 0):
    """Generalized expansion W'(KH, KW', F*C, r*Co) for KW > 1, stride, padding (Appendix A)."""
    wt, host = _as_tensor(w, torch.float32)
    shape = _core.folded_filter_shape(list(wt.shape), factor, stride_w, pad_w)
    out = torch.empty(tuple(shape), dtype=torch.float32, device=wt.device)
    _core.expand_filter_folded(wt.data_ptr(), list(wt.shape), factor, stride_w, pad_w, out.data_ptr(),
                               _stream(wt.device))
    return _ret(out, host)


def replicate_bias(b, factor: int):
    """b'[f*Co + c] = b[c] (src/fold.cpp:213-226), on device."""
    _check_factor(factor)
    bt, host = _as_tensor(b, torch.float32)
    if bt.dim() != 1:
        raise ShapeMismatchError(f"bias must be rank-1, got {tuple(bt.shape)}")
    out = torch.empty(bt.shape[0] * factor, dtype=torch.float32, device=bt.device)
    _core.replicate_bias(bt.data_ptr(), bt.shape[0], factor, out.data_ptr(), _stream(bt.device))
    return _ret(out, host)


def _fold_with_guard(x, w, b, factor, single_channel: bool):
    _check_factor(factor)
    xt, host = _as_tensor(x)
    wt, _ = _as_tensor(w)
    bt, _ = _as_tensor(b)
    if xt.dim() != 4:
        raise ShapeMismatchError(f"apply_width_fold input must be rank-4 NHWC, got {tuple(xt.shape)}")
    if wt.dim() != 4:
        raise ShapeMismatchError(f"apply_width_fold filter must be rank-4, got {tuple(wt.shape)}")
    if bt.dim() != 1 or bt.shape[0] != wt.shape[3]:
        raise ShapeMismatchError(f"bias {tuple(bt.shape)} does not match filter Cout {wt.shape[3]}")
    if xt.shape[3] != wt.shape[2]:
        raise ShapeMismatchError(f"input Cin {xt.shape[3]} != filter Cin {wt.shape[2]}")
    B, H, W, C = xt.shape
    KH, KW, _, Co = wt.shape

    def fallback(reason):
        plan = {"status": "fallback", "reason": reason, "factor": factor, "folded_input_shape": [],
                "expanded_filter_shape": []}
        return plan, _ret(xt, host), _ret(wt, host), _ret(bt, host)

    if W % factor:
        return fallback("WidthNotDivisible")
    if single_channel and C != 1:
        return fallback("UnsupportedChannels")
    if KW != 1:
        return fallback("KernelSpansFoldAxis")
    plan = {"status": "apply", "reason": "None", "factor": factor,
            "folded_input_shape": [B, H, W // factor, C * factor],
            "expanded_filter_shape": [KH, KW, C * factor, factor * Co]}
    x_f = fold_input(xt, factor) if single_channel else fold_input_general(xt, factor)
    return plan, _ret(x_f, host), _ret(expand_filter_general(wt, factor), host), _ret(replicate_bias(bt, factor), host)


def apply_width_fold(x, w, b, factor: int):
    """Algorithm 1 with total fallback, Cin == 1 form (src/fold.cpp:263-309)."""
    return _fold_with_guard(x, w, b, factor, single_channel=True)


def apply_width_fold_general(x, w, b, factor: int, *, stride_w: int | None = None, padding=None,
                             generalized: bool = False):
    """General-Cin fold (src/fold.cpp:311-317). ``generalized=True`` lifts the
    reference's KW == 1 / stride 1 rule and returns the
    dense W'(KH, KW', F*C, r*Co) and b'(r*Co) for that geometry."""
    if not generalized:
        return _fold_with_guard(x, w, b, factor, single_channel=False)
    _check_factor(factor)
    xt, host = _as_tensor(x)
    wt, _ = _as_tensor(w, torch.float32)
    bt, _ = _as_tensor(b, torch.float32)
    sw = int(stride_w or 1)
    ph, pw = _pair(padding or 0)
    B, H, W, C = xt.shape
    KH, KW, _, Co = wt.shape
    if W % factor:
        return ({"status": "fallback", "reason": "WidthNotDivisible", "factor": factor, "folded_input_shape": [],
                 "expanded_filter_shape": []}, _ret(xt, host), _ret(wt, host), _ret(bt, host))
    if factor % sw:
        return ({"status": "fallback", "reason": "StrideOnFoldAxis", "factor": factor, "folded_input_shape": [],
                 "expanded_filter_shape": []}, _ret(xt, host), _ret(wt, host), _ret(bt, host))
    w_f = expand_filter_folded(wt, factor, sw, pw)
    plan = {"status": "apply", "reason": "None", "factor": factor,
            "folded_input_shape": [B, H, W // factor, C * factor], "expanded_filter_shape": list(w_f.shape)}
    return plan, _ret(fold_input_general(xt, factor), host), _ret(w_f, host), _ret(
        replicate_bias(bt, factor // sw), host)


def grouped_conv(x, w_dense, groups: int, stride_h: int = 1, stride_w: int = 1):
    """Verified block-diagonal filter run as groups (src/blockdiag.cpp:138-187).

    Strict-zero check on the device (NotBlockDiagonalError), then the
    exact-order conv in grouped mode (only the diagonal blocks are read, off-block
    terms are never formed) -- bitwise equal to the dense conv2d on finite data,
    as the reference guarantees.
    """
    xt, host = _as_tensor(x, torch.float32)
    wt, _ = _as_tensor(w_dense, torch.float32)
    if wt.dim() != 4:
        raise ShapeMismatchError(f"expanded filter must be rank-4, got {tuple(wt.shape)}")
    scratch = torch.empty(1, dtype=torch.int64, device=wt.device)
    _core.check_block_diagonal(wt.data_ptr(), list(wt.shape), groups, scratch.data_ptr(), _stream(wt.device))
    if xt.dim() != 4:
        raise ShapeMismatchError(f"grouped_conv input must be rank-4 NHWC, got {tuple(xt.shape)}")
    B, H, W, _ = xt.shape
    KH, KW, _, Co = wt.shape
    y = torch.empty((B, max((H - KH) // stride_h + 1, 0), max((W - KW) // stride_w + 1, 0), Co),
                    dtype=torch.float32, device=xt.device)
    _core.conv2d_grouped(xt.data_ptr(), wt.data_ptr(), y.data_ptr(), list(xt.shape), list(wt.shape), stride_h,
                         stride_w, groups, _stream(xt.device))
    return _ret(y, host)


def gemm_ref(a, b):
    """C = A @ B with k innermost (src/gemm.cpp:26-41) via the exact 1x1 conv."""
    at, host = _as_tensor(a, torch.float32)
    bt, _ = _as_tensor(b, torch.float32)
    if at.dim() != 2 or bt.dim() != 2 or at.shape[1] != bt.shape[0]:
        raise ShapeMismatchError(f"gemm shapes {tuple(at.shape)} x {tuple(bt.shape)} do not chain")
    M, K = at.shape
    N = bt.shape[1]
    y = conv2d(at.reshape(1, 1, M, K), bt.reshape(1, 1, K, N), precision="exact")
    return _ret(y.reshape(M, N), host)


def _gemm_operands(a, b, precision):
    dtype = torch.float32 if precision in (None, "exact") else _PREC_DTYPE[precision]
    at, host = _as_tensor(a, dtype)
    bt, _ = _as_tensor(b, dtype)
    if at.dim() != 2 or bt.dim() != 2 or at.shape[1] != bt.shape[0]:
        raise ShapeMismatchError(f"gemm shapes {tuple(at.shape)} x {tuple(bt.shape)} do not chain")
    return at.contiguous(), bt.contiguous(), host, dtype


def gemm_as_conv1x1(a, b, *, precision: str | None = None, out_dtype: torch.dtype | None = None):
    """GEMM as a 1x1 conv over a (1,M,1,K) tensor (src/gemm.cpp:43-49).

    ``precision=None`` is the reference's exact k-inner fp32 order (bitwise
    gemm_ref). ``"bf16"``/``"f16"`` run the UNFOLDED variant of the tcgen05
    kernel (M row = output pixel = GEMM row), the baseline fold_tall_skinny beats.
    """
    if precision in (None, "exact"):
        return gemm_ref(a, b)
    at, bt, host, dtype = _gemm_operands(a, b, precision)
    M, K = at.shape
    N = bt.shape[1]
    fc = FoldedConv2d(bt.reshape(1, 1, K, N), None, (1, M, 1, K), dtype=dtype, variant="unfolded")
    y = fc(at.reshape(1, M, 1, K), bias=False, out_dtype=out_dtype)
    return _ret(y.reshape(M, N), host)


def fold_tall_skinny(a, b, factor: int, *, precision: str | None = None, out_dtype: torch.dtype | None = None):
    """GEMM through a width-folded 1x1 conv (src/gemm.cpp:51-69).

    A (M,K) is read as (1, M/F, F, K) and width-folded into (1, M/F, 1, F*K)
    -- one row-major reshape, zero-copy on the device -- against the
    block-diagonal expansion of B; C is the reshaped folded output.
    ``precision=None`` evaluates it with the reference's exact fp32 conv
    (bitwise = gemm_ref); ``"bf16"``/``"f16"``/``"tf32"`` run the folded
    tcgen05 kernel with fold factor F (the expansion is packed once; C is
    written straight into (M, N) row-major). Raises IllegalFoldError if
    M % F != 0 (src/gemm.cpp:56-60).
    """
    _check_factor(factor)
    at, bt, host, dtype = _gemm_operands(a, b, precision)
    M, K = at.shape
    N = bt.shape[1]
    if M % factor:
        raise IllegalFoldError(f"rows {M} not divisible by {factor}")
    if precision not in (None, "exact"):
        fc = FoldedConv2d(bt.reshape(1, 1, K, N), None, (1, M // factor, factor, K), dtype=dtype, fold=factor)
        y = fc(at.reshape(1, M // factor, factor, K), bias=False, out_dtype=out_dtype)
        return _ret(y.reshape(M, N), host)
    x_f = at.reshape(1, M // factor, 1, K * factor)  # (M,K) as (1,M/F,F,K), width-folded: one reshape
    w_f = expand_filter_general(bt.reshape(1, 1, K, N), factor)
    y_f = conv2d(x_f, w_f, precision="exact")
    return _ret(reconstruct_output(y_f, factor).reshape(M, N), host)


# ------------------------------------------------ graph pass + interpreter (8.F-2)
class Graph:
    """The reference mini-IR (include/widthfold/graph.hpp:21-45) as node dicts
    (``id``, ``op``, ``inputs``, ``shape``, ``tensor``, ``stride_h/w``,
    ``groups``, ``pad_h/w``; ``folded_conv2d`` adds ``factor``, ``bias``) and
    float32 weights. The pass and the interpreter run in the C++ host layer."""

    def __init__(self, nodes=None, weights=None):
        self.nodes = [dict(n) for n in (nodes or [])]
        self.weights = {k: np.ascontiguousarray(v, dtype=np.float32) for k, v in (weights or {}).items()}

    def add(self, id, op, inputs=(), **attrs):
        self.nodes.append({"id": id, "op": op, "inputs": list(inputs), **attrs})
        return id

    def constant(self, id, array):
        self.weights[id] = np.ascontiguousarray(array, dtype=np.float32)
        return self.add(id, "constant", tensor=id)

    def infer_shapes(self) -> "Graph":
        return Graph(_core.infer_shapes(self.nodes, self.weights), self.weights)

    def find(self, id):
        return next((n for n in self.nodes if n["id"] == id), None)


def width_fold_pass(graph: Graph, factor: int | None = None, align: int = 8, precision: str = "tf32"):
    """Rewrite every conv2d the generalized device fold applies to into one
    ``folded_conv2d`` (tcgen05; sole-consumer constant bias fused).
    ``precision``: "tf32" (default, within 1e-3 of the f32 graph) or
    "bf16"/"f16" (the node casts its input and filter on the device; 1e-2).
    Returns ``(graph, report)`` like PassResult (include/widthfold/pass.hpp:45-52)."""
    nodes, weights, report = _core.width_fold_pass(graph.nodes, graph.weights, int(factor or 0), int(align),
                                                   {"fp16": "f16"}.get(precision, precision))
    return Graph(nodes, weights), report


def interpret(graph: Graph, inputs: dict, mode: str = "device") -> dict:
    """Execute on the GPU; returns {output id: float32 ndarray} (src/interpreter.cpp:8-66)."""
    if mode not in ("dense", "grouped", "device"):
        raise ValueError("mode must be 'dense', 'grouped' or 'device'")
    arrays = {k: np.ascontiguousarray(np.asarray(v, dtype=np.float32)) for k, v in inputs.items()}
    return _core.interpret(graph.nodes, graph.weights, arrays, mode)


ShapeInferenceFailureError = _core.ShapeInferenceFailureError
MissingInputError = _core.MissingInputError


# ------------------------------------------- model format: bundles + graph JSON (8.F-4)
ManifestParseError = _core.ManifestParseError
BlobSizeMismatchError = _core.BlobSizeMismatchError
IoFailureError = _core.IoFailureError


def read_bundle(manifest_path) -> dict:
    """Tensor bundle (manifest + raw little-endian blobs, docs/model_format.md;
    include/widthfold/bundle.hpp:32-36) -> {name: array} in manifest order.
    ``f32``/``f16`` come back as numpy arrays, ``bf16`` as CPU torch tensors;
    bit patterns (signed zeros, subnormals, NaN payloads) are preserved."""
    out = {}
    for name, shape, dtype, raw in _core.read_bundle(str(manifest_path)):
        if dtype == "bf16":
            bits = np.frombuffer(raw, dtype="<u2").astype(np.int16).reshape(shape)
            out[name] = torch.from_numpy(bits.copy()).view(torch.bfloat16)
        else:
            out[name] = np.frombuffer(raw, dtype="<f4" if dtype == "f32" else "<f2").reshape(shape).copy()
    return out


def _bundle_entry(name, v):
    if isinstance(v, torch.Tensor):
        v = v.detach().cpu().contiguous()
        if v.dtype == torch.bfloat16:
            return (name, list(v.shape), "bf16", v.view(torch.int16).numpy().astype("<i2").tobytes())
        v = v.numpy()
    a = np.ascontiguousarray(v)
    if a.dtype == np.float16:
        return (name, list(a.shape), "f16", a.astype("<f2").tobytes())
    if a.dtype != np.float32:
        a = a.astype(np.float32)
    return (name, list(a.shape), "f32", a.astype("<f4").tobytes())


def write_bundle(manifest_path, tensors: dict) -> None:
    """Write ``tensors`` ({name: array}; float32 / float16 numpy or torch, or
    torch bfloat16) as a manifest plus ``<stem>.bin`` (bundle.hpp:38-40)."""
    _core.write_bundle(str(manifest_path), [_bundle_entry(k, v) for k, v in tensors.items()])


def read_graph(path) -> Graph:
    """Graph JSON + its weights bundle (include/widthfold/graph.hpp:68-70); the
    constants load as float32 graph values whatever their bundle dtype."""
    nodes, weights = _core.read_graph(str(path))
    return Graph(nodes, weights)


def write_graph(graph: Graph, path) -> None:
    """Graph JSON plus ``<stem>.weights.json``/``.bin`` beside it (src/graph.cpp:315-339)."""
    _core.write_graph(graph.nodes, graph.weights, str(path))

__all__ = [
    "apply_width_fold", "apply_width_fold_general", "bias_add", "check_legality", "choose_fold_factor",
    "conv1d_h", "conv2d", "count_macs", "expand_filter", "expand_filter_general", "fold_input",
    "fold_input_general", "fold_tall_skinny", "gemm_as_conv1x1", "gemm_ref", "grouped_conv", "mac_report",
    "reconstruct_output", "replicate_bias", "unfold_input_general",
    # additions
    "FoldedConv2d", "expand_filter_folded", "plan_fold", "ShapeMismatchError", "IllegalFoldError",
    "DegenerateOutputError", "NotBlockDiagonalError", "UnsupportedError",
    "Graph", "width_fold_pass", "interpret", "ShapeInferenceFailureError", "MissingInputError",
    "read_bundle", "write_bundle", "read_graph", "write_graph", "ManifestParseError", "BlobSizeMismatchError",
    "IoFailureError",
]
