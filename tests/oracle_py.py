"""numpy face of oracle/liboracle.so -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use this.
Each method calls the plain-C restatement in oracle/oracle.c, which cites the
reference file:line it follows.
"""
import ctypes

import numpy as np

_f = ctypes.POINTER(ctypes.c_float)
_i = ctypes.c_int64


def _p(a):
    return a.ctypes.data_as(_f)


class Oracle:
    def __init__(self, lib):
        self.lib = lib
        for name in ("or_conv2d", "or_bias_add", "or_relu", "or_pad_nhwc", "or_fold_input_general",
                     "or_unfold_input_general", "or_expand_filter_general", "or_replicate_bias",
                     "or_reconstruct_output", "or_grouped_conv", "or_expand_filter_folded", "or_conv_folded",
                     "or_fold_geometry"):
            getattr(lib, name).restype = None
        lib.or_count_macs.restype = ctypes.c_uint64

    def conv2d(self, x, w, sh=1, sw=1):
        x = np.ascontiguousarray(x, np.float32)
        w = np.ascontiguousarray(w, np.float32)
        B, H, W, C = x.shape
        KH, KW, _, Co = w.shape
        OH, OW = (H - KH) // sh + 1, (W - KW) // sw + 1
        y = np.empty((B, OH, OW, Co), np.float32)
        self.lib.or_conv2d(_p(x), _i(B), _i(H), _i(W), _i(C), _p(w), _i(KH), _i(KW), _i(Co), _i(sh), _i(sw), _p(y))
        return y

    def bias_add(self, y, b):
        y = np.array(y, np.float32, copy=True)
        b = np.ascontiguousarray(b, np.float32)
        self.lib.or_bias_add(_p(y), _i(y.size), _p(b), _i(b.size))
        return y

    def relu(self, y):
        y = np.array(y, np.float32, copy=True)
        self.lib.or_relu(_p(y), _i(y.size))
        return y

    def pad(self, x, ph, pw):
        x = np.ascontiguousarray(x, np.float32)
        B, H, W, C = x.shape
        xp = np.empty((B, H + 2 * ph, W + 2 * pw, C), np.float32)
        self.lib.or_pad_nhwc(_p(x), _i(B), _i(H), _i(W), _i(C), _i(ph), _i(pw), _p(xp))
        return xp

    def conv_padded(self, x, w, b, stride, pad, relu=False):
        """The reference way to evaluate a padded conv: explicit zero pad + VALID conv2d + bias_add (+ReLU)."""
        y = self.conv2d(self.pad(x, pad, pad), w, stride, stride)
        if b is not None:
            y = self.bias_add(y, b)
        return self.relu(y) if relu else y

    def fold_input_general(self, x, F):
        x = np.ascontiguousarray(x, np.float32)
        B, H, W, C = x.shape
        out = np.empty((B, H, W // F, C * F), np.float32)
        self.lib.or_fold_input_general(_p(x), _i(B), _i(H), _i(W), _i(C), _i(F), _p(out))
        return out

    def unfold_input_general(self, xf, F):
        xf = np.ascontiguousarray(xf, np.float32)
        B, H, Wf, Cf = xf.shape
        out = np.empty((B, H, Wf * F, Cf // F), np.float32)
        self.lib.or_unfold_input_general(_p(xf), _i(B), _i(H), _i(Wf), _i(Cf), _i(F), _p(out))
        return out

    def expand_filter_general(self, w, F):
        w = np.ascontiguousarray(w, np.float32)
        KH, KW, C, Co = w.shape
        assert KW == 1
        out = np.empty((KH, 1, C * F, Co * F), np.float32)
        self.lib.or_expand_filter_general(_p(w), _i(KH), _i(C), _i(Co), _i(F), _p(out))
        return out

    def replicate_bias(self, b, F):
        b = np.ascontiguousarray(b, np.float32)
        out = np.empty(b.size * F, np.float32)
        self.lib.or_replicate_bias(_p(b), _i(b.size), _i(F), _p(out))
        return out

    def reconstruct_output(self, y, F):
        y = np.ascontiguousarray(y, np.float32)
        B, H, Wf, Cf = y.shape
        out = np.empty((B, H, Wf * F, Cf // F), np.float32)
        self.lib.or_reconstruct_output(_p(y), _i(B), _i(H), _i(Wf), _i(Cf), _i(F), _p(out))
        return out

    def grouped_conv(self, x, wd, F, sh=1, sw=1):
        x = np.ascontiguousarray(x, np.float32)
        wd = np.ascontiguousarray(wd, np.float32)
        B, H, W, Cif = x.shape
        KH, KW, _, Cof = wd.shape
        y = np.empty((B, (H - KH) // sh + 1, (W - KW) // sw + 1, Cof), np.float32)
        self.lib.or_grouped_conv(_p(x), _i(B), _i(H), _i(W), _i(Cif), _p(wd), _i(KH), _i(KW), _i(Cof), _i(F),
                                 _i(sh), _i(sw), _p(y))
        return y

    def fold_geometry(self, f, s, pw, KW):
        r, c0, kwf = _i(0), _i(0), _i(0)
        self.lib.or_fold_geometry(_i(f), _i(s), _i(pw), _i(KW), ctypes.byref(r), ctypes.byref(c0), ctypes.byref(kwf))
        return r.value, c0.value, kwf.value

    def expand_filter_folded(self, w, f, s, pw):
        w = np.ascontiguousarray(w, np.float32)
        KH, KW, C, Co = w.shape
        r, c0, kwf = self.fold_geometry(f, s, pw, KW)
        out = np.empty((KH, kwf, f * C, r * Co), np.float32)
        self.lib.or_expand_filter_folded(_p(w), _i(KH), _i(KW), _i(C), _i(Co), _i(f), _i(s), _i(pw), _p(out))
        return out

    def conv_folded(self, x, wexp, KH, KW, Co, f, s, ph, pw):
        x = np.ascontiguousarray(x, np.float32)
        wexp = np.ascontiguousarray(wexp, np.float32)
        B, H, W, C = x.shape
        OH, OW = (H + 2 * ph - KH) // s + 1, (W + 2 * pw - KW) // s + 1
        y = np.zeros((B, OH, OW, Co), np.float32)
        self.lib.or_conv_folded(_p(x), _i(B), _i(H), _i(W), _i(C), _p(wexp), _i(KH), _i(KW), _i(Co), _i(f), _i(s),
                                _i(ph), _i(pw), _p(y))
        return y

    def count_macs(self, B, OH, OW, Co, KH, KW, C):
        return int(self.lib.or_count_macs(_i(B), _i(OH), _i(OW), _i(Co), _i(KH), _i(KW), _i(C)))
