"""fp64 CPU oracle for the conv2d operator -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline
leg may import this module.  It shares no code with the CUDA path.

Three independent formulations of the same definition ("2D
convolution" operator; "RELU operator"; output invariance P:381; the
written-out definition is SURVEY.md 8(c)):

* ``conv2d_c``      -- the C fp64 direct loop in ``conv_oracle.c`` (OpenMP over
                       (n, k)); this is the one timed as the CPU baseline.
* ``conv2d_numpy``  -- numpy fp64: ``np.pad`` + ``sliding_window_view`` +
                       ``einsum`` (a library contraction as one step).
* ``conv2d_brute``  -- pure-Python loops, tiny shapes only.

Inputs are logical NCHW (x), KCRS = (K, C/g, R, S) (w), (K,) (bias); the
output is NKPQ.  Readings C1-C5, C9: cross-correlation, symmetric
zero padding, floor output formula, dilation >= 1, groups dividing C and K,
bias then ReLU.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "conv_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


class OracleDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "n", "c", "h", "w", "k", "r", "s",
        "stride_h", "stride_w", "pad_h", "pad_w", "dil_h", "dil_w", "groups",
        "has_bias", "relu")]


def build(force: bool = False) -> str:
    """Compile conv_oracle.c into liboracle.so (gcc, -O2, OpenMP, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fopenmp", "-fPIC", "-shared",
                               "-fno-fast-math", "-o", tmp, _SRC])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P = ctypes.POINTER
            lib.oracle_out_dim.argtypes = [ctypes.c_int32] * 5
            lib.oracle_out_dim.restype = ctypes.c_int
            lib.oracle_conv2d_f64.argtypes = [P(OracleDesc), ctypes.c_void_p, ctypes.c_void_p,
                                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
            lib.oracle_conv2d_f64.restype = ctypes.c_int
            lib.oracle_conv2d_points_f64.argtypes = [P(OracleDesc), ctypes.c_void_p, ctypes.c_void_p,
                                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                                     ctypes.c_void_p, ctypes.c_int32]
            lib.oracle_conv2d_points_f64.restype = ctypes.c_int
            lib.oracle_max_threads.restype = ctypes.c_int
            _lib = lib
    return _lib


def out_dim(n_in: int, k: int, stride: int, pad: int, dil: int = 1) -> int:
    """P = floor((H + 2 pad - dil (R-1) - 1) / stride) + 1, via the C oracle."""
    return int(_load().oracle_out_dim(n_in, k, stride, pad, dil))


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def _desc(shape: dict, has_bias: bool, relu: bool) -> OracleDesc:
    g = shape.get
    return OracleDesc(g("n"), g("c"), g("h"), g("w"), g("k"), g("r"), g("s"),
                      g("stride_h", g("stride", 1)), g("stride_w", g("stride", 1)),
                      g("pad_h", g("pad", 0)), g("pad_w", g("pad", 0)),
                      g("dil_h", g("dil", 1)), g("dil_w", g("dil", 1)), g("groups", 1),
                      int(has_bias), int(relu))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def conv2d_c(shape: dict, x, w, bias=None, relu: bool = False, threads: int = 0) -> np.ndarray:
    """Full NKPQ output via the C fp64 loop. ``shape`` keys: n c h w k r s
    stride[_h/_w] pad[_h/_w] dil[_h/_w] groups."""
    d = _desc(shape, bias is not None, relu)
    x, w = _f64(x), _f64(w)
    b = _f64(bias) if bias is not None else np.zeros(1)
    P = out_dim(d.h, d.r, d.stride_h, d.pad_h, d.dil_h)
    Q = out_dim(d.w, d.s, d.stride_w, d.pad_w, d.dil_w)
    if P < 1 or Q < 1:
        raise ValueError("invalid conv shape (P or Q < 1)")
    assert x.shape == (d.n, d.c, d.h, d.w), x.shape
    assert w.shape == (d.k, d.c // d.groups, d.r, d.s), w.shape
    y = np.empty((d.n, d.k, P, Q), dtype=np.float64)
    rc = _load().oracle_conv2d_f64(ctypes.byref(d), x.ctypes.data, w.ctypes.data, b.ctypes.data,
                                   y.ctypes.data, threads)
    if rc != 0:
        raise ValueError(f"oracle rejected descriptor (rc={rc})")
    return y


def conv2d_points_c(shape: dict, x, w, bias, relu: bool, flat_idx, threads: int = 0) -> np.ndarray:
    """Selected outputs (flat NKPQ indices) via the C fp64 loop."""
    d = _desc(shape, bias is not None, relu)
    x, w = _f64(x), _f64(w)
    b = _f64(bias) if bias is not None else np.zeros(1)
    idx = np.ascontiguousarray(flat_idx, dtype=np.int64)
    out = np.empty(idx.shape[0], dtype=np.float64)
    rc = _load().oracle_conv2d_points_f64(ctypes.byref(d), x.ctypes.data, w.ctypes.data,
                                          b.ctypes.data, idx.ctypes.data, idx.shape[0],
                                          out.ctypes.data, threads)
    if rc != 0:
        raise ValueError(f"oracle rejected points (rc={rc})")
    return out


def conv2d_numpy(shape: dict, x, w, bias=None, relu: bool = False) -> np.ndarray:
    """Independent numpy fp64 formulation: zero-pad, take every (dil-spaced)
    R x S window at stride, contract over (c', r, s) per group with einsum."""
    g = shape.get
    n, c, h, wd, k, r, s = (g(a) for a in ("n", "c", "h", "w", "k", "r", "s"))
    sh, sw = g("stride_h", g("stride", 1)), g("stride_w", g("stride", 1))
    ph, pw = g("pad_h", g("pad", 0)), g("pad_w", g("pad", 0))
    dh, dw = g("dil_h", g("dil", 1)), g("dil_w", g("dil", 1))
    groups = g("groups", 1)
    x, w = _f64(x), _f64(w)
    xp = np.pad(x, ((0, 0), (0, 0), (ph, ph), (pw, pw)))
    eh, ew = dh * (r - 1) + 1, dw * (s - 1) + 1          # dilated window extent
    win = np.lib.stride_tricks.sliding_window_view(xp, (eh, ew), axis=(2, 3))
    win = win[:, :, ::sh, ::sw, ::dh, ::dw]               # (N, C, P, Q, R, S)
    cg, kg = c // groups, k // groups
    outs = []
    for gi in range(groups):
        xs = win[:, gi * cg:(gi + 1) * cg]
        ws = w[gi * kg:(gi + 1) * kg]
        outs.append(np.einsum("ncpqrs,kcrs->nkpq", xs, ws, optimize=True))
    y = np.concatenate(outs, axis=1)
    if bias is not None:
        y = y + _f64(bias)[None, :, None, None]
    if relu:
        y = np.maximum(y, 0.0)
    return y


def conv2d_brute(shape: dict, x, w, bias=None, relu: bool = False) -> np.ndarray:
    """Pure-Python loops over the definition; tiny shapes only."""
    g = shape.get
    n, c, h, wd, k, r, s = (g(a) for a in ("n", "c", "h", "w", "k", "r", "s"))
    sh, sw = g("stride_h", g("stride", 1)), g("stride_w", g("stride", 1))
    ph, pw = g("pad_h", g("pad", 0)), g("pad_w", g("pad", 0))
    dh, dw = g("dil_h", g("dil", 1)), g("dil_w", g("dil", 1))
    groups = g("groups", 1)
    # Window origins counted by enumeration, not by the closed form.
    P = sum(1 for o in range(-ph, h + ph) if (o + ph) % sh == 0 and o + dh * (r - 1) <= h - 1 + ph)
    Q = sum(1 for o in range(-pw, wd + pw) if (o + pw) % sw == 0 and o + dw * (s - 1) <= wd - 1 + pw)
    cg, kg = c // groups, k // groups
    xl, wl = np.asarray(x, dtype=np.float64).tolist(), np.asarray(w, dtype=np.float64).tolist()
    y = np.zeros((n, k, P, Q))
    for ni in range(n):
        for ki in range(k):
            c0 = (ki // kg) * cg
            for p in range(P):
                for q in range(Q):
                    acc = 0.0
                    for cc in range(cg):
                        for ri in range(r):
                            hi = p * sh - ph + ri * dh
                            if not 0 <= hi < h:
                                continue
                            for si in range(s):
                                wi = q * sw - pw + si * dw
                                if 0 <= wi < wd:
                                    acc += xl[ni][c0 + cc][hi][wi] * wl[ki][cc][ri][si]
                    if bias is not None:
                        acc += float(bias[ki])
                    if relu and acc < 0:
                        acc = 0.0
                    y[ni, ki, p, q] = acc
    return y
