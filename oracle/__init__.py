"""CPU oracle for the Caffe convolution hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_1408_5093_b200``) never imports it, and this package never imports the
product path: they share no code, headers, tables or constants.

Loop-nest definitions live in ``oracle.c`` (plain C, fp64 accumulation, built by
``build()`` with ``gcc -O2 -ffp-contract=off -fopenmp``).  The small dense ops
(inner product, ReLU, softmax loss, SGD) are written here in numpy; a matmul is
allowed as a library step.  Every function cites the passage it follows
(``P:n`` = /root/reference/PAPER.md line, ``S:n`` = SPEC.md line, ``Rn`` =
DESIGN.md reading).

Parity pins for every function are in ``tests/test_oracle_*.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (plain gcc, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
               "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


def _L():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
        d, f, i, i32p = (ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_float),
                         ctypes.c_int, ctypes.POINTER(ctypes.c_int32))
        dbl = ctypes.c_double
        _lib.oracle_conv_out_dim.argtypes = [i, i, i, i]
        _lib.oracle_pool_out_dim.argtypes = [i, i, i, i]
        _lib.oracle_conv_forward.argtypes = [d, d, d] + [i] * 13 + [d]
        _lib.oracle_conv_backward_data.argtypes = [d, d] + [i] * 12 + [dbl, d]
        _lib.oracle_conv_backward_weight.argtypes = [d, d] + [i] * 12 + [dbl, d, d]
        _lib.oracle_im2col_f32.argtypes = [f] + [i] * 10 + [f]
        _lib.oracle_col2im_f32.argtypes = [f] + [i] * 10 + [f]
        _lib.oracle_maxpool_forward_f32.argtypes = [f] + [i] * 10 + [f, i32p]
        _lib.oracle_maxpool_backward_f32.argtypes = [f, i32p] + [i] * 10 + [f]
        _lib.oracle_maxpool_forward_f64.argtypes = [d] + [i] * 10 + [d, i32p]
        _lib.oracle_maxpool_backward_f64.argtypes = [d, i32p] + [i] * 10 + [d]
        _lib.oracle_avepool_forward.argtypes = [d] + [i] * 10 + [d]
        _lib.oracle_avepool_backward.argtypes = [d] + [i] * 10 + [d]
        _lib.oracle_lrn_forward.argtypes = [d] + [i] * 5 + [dbl] * 3 + [d, d]
        _lib.oracle_lrn_backward.argtypes = [d, d] + [i] * 5 + [dbl] * 3 + [d]
    return _lib


def _pd(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _pf(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def _pi(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


# ----------------------------------------------------------------------------- shapes
def conv_out_dim(n: int, k: int, s: int, p: int) -> int:
    """S:122 floor rule."""
    return _L().oracle_conv_out_dim(n, k, s, p)


def pool_out_dim(n: int, k: int, s: int, p: int) -> int:
    """S:126 ceil rule, clipped per reading R5."""
    return _L().oracle_pool_out_dim(n, k, s, p)


# ----------------------------------------------------------------------------- conv
def conv_forward(X, W, b=None, stride=(1, 1), pad=(0, 0), group=1, relu=False):
    """S:145 (+groups R3, fused ReLU S:199).  X (N,C,H,W), W (O,C/g,kh,kw), b (O,) -> fp64 Y."""
    X, W = _f64(X), _f64(W)
    N, C, H, Wd = X.shape
    O, Cg, kh, kw = W.shape
    assert Cg * group == C and O % group == 0
    OH, OW = conv_out_dim(H, kh, stride[0], pad[0]), conv_out_dim(Wd, kw, stride[1], pad[1])
    Y = np.empty((N, O, OH, OW), np.float64)
    bb = _f64(b) if b is not None else None
    _L().oracle_conv_forward(_pd(X), _pd(W), _pd(bb) if bb is not None else None,
                             N, C, H, Wd, O, kh, kw, stride[0], stride[1], pad[0], pad[1],
                             group, int(bool(relu)), _pd(Y))
    return Y


def conv_backward_data(dY, W, in_shape, stride=(1, 1), pad=(0, 0), group=1, beta=0.0, dX=None):
    """S:154 data gradient (exact adjoint of S:145).  Returns fp64 dX of in_shape."""
    dY, W = _f64(dY), _f64(W)
    N, C, H, Wd = in_shape
    O, Cg, kh, kw = W.shape
    out = np.zeros(in_shape, np.float64) if dX is None else _f64(dX).copy()
    _L().oracle_conv_backward_data(_pd(dY), _pd(W), N, C, H, Wd, O, kh, kw, stride[0], stride[1],
                                   pad[0], pad[1], group, float(beta), _pd(out))
    return out


def conv_backward_weight(X, dY, w_shape, stride=(1, 1), pad=(0, 0), group=1, beta=0.0,
                         dW=None, db=None):
    """S:154 weight/bias gradient, accumulate via beta (R4).  Returns (dW, db) fp64."""
    X, dY = _f64(X), _f64(dY)
    N, C, H, Wd = X.shape
    O, Cg, kh, kw = w_shape
    dWo = np.zeros(w_shape, np.float64) if dW is None else _f64(dW).copy()
    dbo = np.zeros((O,), np.float64) if db is None else _f64(db).copy()
    _L().oracle_conv_backward_weight(_pd(X), _pd(dY), N, C, H, Wd, O, kh, kw, stride[0], stride[1],
                                     pad[0], pad[1], group, float(beta), _pd(dWo), _pd(dbo))
    return dWo, dbo


def im2col(X, n, ksize, stride=(1, 1), pad=(0, 0)):
    """S:297/S:806 patch matrix for image n: (C*kh*kw, OH*OW) float32, bit-exact data movement."""
    X = _f32(X)
    N, C, H, Wd = X.shape
    kh, kw = ksize
    OH, OW = conv_out_dim(H, kh, stride[0], pad[0]), conv_out_dim(Wd, kw, stride[1], pad[1])
    col = np.empty((C * kh * kw, OH * OW), np.float32)
    _L().oracle_im2col_f32(_pf(X), n, C, H, Wd, kh, kw, stride[0], stride[1], pad[0], pad[1], _pf(col))
    return col


def col2im(col, in_shape, n, ksize, stride=(1, 1), pad=(0, 0), out=None):
    """Adjoint of im2col with fixed FP32 gather order; writes image n of out (float32)."""
    col = _f32(col)
    N, C, H, Wd = in_shape
    kh, kw = ksize
    dX = np.zeros(in_shape, np.float32) if out is None else out
    _L().oracle_col2im_f32(_pf(col), n, C, H, Wd, kh, kw, stride[0], stride[1], pad[0], pad[1], _pf(dX))
    return dX


# ----------------------------------------------------------------------------- pooling
def maxpool_forward(X, ksize, stride, pad=(0, 0), fp64=False):
    """S:163 max with R7 ties/index; (Y, mask int32).  float32 in/out (the bit-exact GPU parity
    form) or, with fp64=True, float64 in/out (oracle/net.py): selection does not round, so both
    pick the same element of the same values."""
    X = _f64(X) if fp64 else _f32(X)
    N, C, H, Wd = X.shape
    OH = pool_out_dim(H, ksize[0], stride[0], pad[0])
    OW = pool_out_dim(Wd, ksize[1], stride[1], pad[1])
    Y = np.empty((N, C, OH, OW), X.dtype)
    M = np.empty((N, C, OH, OW), np.int32)
    fn = _L().oracle_maxpool_forward_f64 if fp64 else _L().oracle_maxpool_forward_f32
    fn(_pd(X) if fp64 else _pf(X), N, C, H, Wd, ksize[0], ksize[1], stride[0], stride[1],
       pad[0], pad[1], _pd(Y) if fp64 else _pf(Y), _pi(M))
    return Y, M


def maxpool_backward(dY, mask, in_shape, ksize, stride, pad=(0, 0), fp64=False):
    """S:172 routing by argmax, gather in ascending (py,px) order (R8): FP32 sums (the bit-exact
    GPU order) or, with fp64=True, double sums (oracle/net.py)."""
    dY = _f64(dY) if fp64 else _f32(dY)
    mask = np.ascontiguousarray(mask, dtype=np.int32)
    N, C, H, Wd = in_shape
    dX = np.empty(in_shape, dY.dtype)
    fn = _L().oracle_maxpool_backward_f64 if fp64 else _L().oracle_maxpool_backward_f32
    fn(_pd(dY) if fp64 else _pf(dY), _pi(mask), N, C, H, Wd, ksize[0], ksize[1],
       stride[0], stride[1], pad[0], pad[1], _pd(dX) if fp64 else _pf(dX))
    return dX


def avepool_forward(X, ksize, stride, pad=(0, 0)):
    """S:163 window mean with the R6 divisor; fp64."""
    X = _f64(X)
    N, C, H, Wd = X.shape
    OH = pool_out_dim(H, ksize[0], stride[0], pad[0])
    OW = pool_out_dim(Wd, ksize[1], stride[1], pad[1])
    Y = np.empty((N, C, OH, OW), np.float64)
    _L().oracle_avepool_forward(_pd(X), N, C, H, Wd, ksize[0], ksize[1], stride[0], stride[1],
                                pad[0], pad[1], _pd(Y))
    return Y


def avepool_backward(dY, in_shape, ksize, stride, pad=(0, 0)):
    """S:172 uniform spread; exact adjoint of avepool_forward; fp64."""
    dY = _f64(dY)
    N, C, H, Wd = in_shape
    dX = np.empty(in_shape, np.float64)
    _L().oracle_avepool_backward(_pd(dY), N, C, H, Wd, ksize[0], ksize[1], stride[0], stride[1],
                                 pad[0], pad[1], _pd(dX))
    return dX


# ----------------------------------------------------------------------------- LRN
def lrn_forward(X, size=5, alpha=1e-4, beta=0.75, k=1.0, want_scale=False):
    """S:217 across-channel LRN, alpha/n scaling, clipped window (R9); fp64."""
    X = _f64(X)
    N, C, H, Wd = X.shape
    Y = np.empty_like(X)
    S = np.empty_like(X) if want_scale else None
    _L().oracle_lrn_forward(_pd(X), N, C, H, Wd, size, alpha, beta, k, _pd(Y),
                            _pd(S) if S is not None else None)
    return (Y, S) if want_scale else Y


def lrn_backward(X, dY, size=5, alpha=1e-4, beta=0.75, k=1.0):
    """S:226 exact gradient of lrn_forward; fp64."""
    X, dY = _f64(X), _f64(dY)
    N, C, H, Wd = X.shape
    dX = np.empty_like(X)
    _L().oracle_lrn_backward(_pd(X), _pd(dY), N, C, H, Wd, size, alpha, beta, k, _pd(dX))
    return dX


# ----------------------------------------------------------------------------- inner product
def ip_forward(X, W, b=None):
    """out[n,k] = bias[k] + sum_d w[k,d] in[n,d]; input flattened to (N, C*H*W)."""
    X = _f64(X).reshape(X.shape[0], -1)
    W = _f64(W).reshape(W.shape[0], -1)
    Y = X @ W.T
    if b is not None:
        Y = Y + _f64(b)[None, :]
    return Y


def ip_backward(X, W, dY):
    """dW[k,d] = sum_n dY[n,k] in[n,d]; dX[n,d] = sum_k dY[n,k] w[k,d]; db[k] = sum_n dY[n,k]."""
    X2 = _f64(X).reshape(X.shape[0], -1)
    W2 = _f64(W).reshape(W.shape[0], -1)
    dY2 = _f64(dY).reshape(dY.shape[0], -1)
    return (dY2 @ W2).reshape(X.shape), dY2.T @ X2, dY2.sum(axis=0)


# ----------------------------------------------------------------------------- ReLU, losses, SGD
def relu_forward(X):
    """max(0, x); the value at x<=0 is +0.0 (R10)."""
    X = np.asarray(X)
    return np.where(X > 0, X, np.zeros_like(X))


def relu_backward(X, dY):
    """dY where x > 0 else 0 (gradient 0 at x == 0)."""
    X, dY = np.asarray(X), np.asarray(dY)
    return np.where(X > 0, dY, np.zeros_like(dY))


def softmax_loss(scores, labels):
    """S:253 loss = -(1/N) sum_n log softmax(s_n)[l_n] (max-subtracted); S:262 diff = (p - 1_l)/N."""
    s = _f64(scores).reshape(scores.shape[0], -1)
    N = s.shape[0]
    z = s - s.max(axis=1, keepdims=True)
    lse = np.log(np.exp(z).sum(axis=1))
    lab = np.asarray(labels).astype(np.int64).reshape(-1)
    loss = float(np.mean(lse - z[np.arange(N), lab]))
    p = np.exp(z - lse[:, None])
    p[np.arange(N), lab] -= 1.0
    return loss, p / N


def sgd_update(w, g, v, lr, momentum, decay, grad_scale=1.0):
    """S:523 (R18 form): g' = g*grad_scale + decay*w; v <- momentum*v - lr*g'; w <- w + v.  fp64."""
    w, g, v = _f64(w), _f64(g), _f64(v)
    gp = g * grad_scale + decay * w
    v2 = momentum * v - lr * gp
    return w + v2, v2


# ----------------------------------------------------------------------------- catalogue layers (NEXT-4)
def sigmoid_forward(X):
    """S:199 logistic nonlinearity ("nonlinearities like rectified linear and logistic"):
    out = 1 / (1 + e^-x); fp64."""
    X = _f64(X)
    return 1.0 / (1.0 + np.exp(-X))


def sigmoid_backward(Y, dY):
    """bottom_diff = top_diff * out * (1 - out), from the forward OUTPUT (the
    in-place sigmoid keeps only its output); fp64."""
    Y, dY = _f64(Y), _f64(dY)
    return dY * Y * (1.0 - Y)


def eltwise_forward(inputs, op, coeffs=None):
    """S:235 element-wise operations: sum = sum_i coeff_i x_i (coeffs default 1), prod =
    prod_i x_i, max = elementwise max; >= 2 inputs of one shape; fp64, inputs
    combined in list order."""
    xs = [_f64(x) for x in inputs]
    if len(xs) < 2:
        raise ValueError("eltwise needs at least 2 inputs (S:236)")
    if any(x.shape != xs[0].shape for x in xs):
        raise ValueError("eltwise inputs must have identical shapes (S:236)")
    if op == "sum":
        c = [1.0] * len(xs) if coeffs is None else [float(v) for v in coeffs]
        out = c[0] * xs[0]
        for ci, x in zip(c[1:], xs[1:]):
            out = out + ci * x
        return out
    if op == "prod":
        out = xs[0].copy()
        for x in xs[1:]:
            out = out * x
        return out
    if op == "max":
        out = xs[0].copy()
        for x in xs[1:]:
            out = np.where(x > out, x, out)
        return out
    raise ValueError(f"unknown eltwise op {op}")


def eltwise_backward(inputs, dY, op, coeffs=None):
    """sum: diff_i = coeff_i dY; prod: diff_i = dY * prod_{j != i} x_j (the product of the
    other inputs, written out -- no division by x_i); max: dY routed to the per-element argmax
    input, the FIRST one on ties.  Returns a list of fp64 diffs."""
    xs = [_f64(x) for x in inputs]
    dY = _f64(dY)
    n = len(xs)
    if op == "sum":
        c = [1.0] * n if coeffs is None else [float(v) for v in coeffs]
        return [ci * dY for ci in c]
    if op == "prod":
        out = []
        for i in range(n):
            p = np.ones_like(dY)
            for j in range(n):
                if j != i:
                    p = p * xs[j]
            out.append(dY * p)
        return out
    if op == "max":
        arg = np.zeros(dY.shape, np.int64)
        best = xs[0].copy()
        for i in range(1, n):
            better = xs[i] > best          # strict: an equal later input never takes the gradient
            arg = np.where(better, i, arg)
            best = np.where(better, xs[i], best)
        return [np.where(arg == i, dY, 0.0) for i in range(n)]
    raise ValueError(f"unknown eltwise op {op}")


def hinge_loss(scores, labels):
    """S:271 one-vs-all L1 hinge ("losses like softmax and hinge"): y_nk = +1 if k = l_n else
    -1; loss = (1/N) sum_{n,k} max(0, 1 - y_nk s_nk); diff_nk = -y_nk [1 - y_nk s_nk > 0] / N.
    Labels outside [0, K) are an error.  Returns (loss, diff) in fp64."""
    s = _f64(scores).reshape(scores.shape[0], -1)
    N, K = s.shape
    lab = np.asarray(labels).astype(np.int64).reshape(-1)
    if lab.shape[0] != N or np.any(lab < 0) or np.any(lab >= K):
        raise ValueError("hinge loss: label out of range (S:273)")
    y = -np.ones_like(s)
    y[np.arange(N), lab] = 1.0
    m = 1.0 - y * s
    loss = float(np.maximum(m, 0.0).sum() / N)
    diff = np.where(m > 0, -y, 0.0) / N
    return loss, diff


# ----------------------------------------------------------------------------- operand quantizers
def quant_bf16(x):
    """Round-to-nearest-even FP32 -> BF16 (reading R12/R14), returned as float32 values."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return (r & 0xFFFFFFFF).astype(np.uint32).view(np.float32).reshape(a.shape)


def quant_tf32_rz(x):
    """TF32 by truncation of the low 13 mantissa bits (reading R12, raw fp32 bits fed to the MMA)."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    return (a.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32).reshape(a.shape)


def quant_tf32_rn(x):
    """TF32 round-to-nearest-even on the 10-bit mantissa (reading R12)."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0xFFF + ((u >> 13) & 1)) >> 13) << 13
    return (r & 0xFFFFFFFF).astype(np.uint32).view(np.float32).reshape(a.shape)
