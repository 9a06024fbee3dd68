"""B200-native Caffe convolution hot path (arXiv 1408.5093) -- thin Python binding.

Every function here only marshals torch CUDA tensors into the C ABI declared in
include/caffe_b200.h (``caffe_*`` entry points of libcaffe_b200.so) and passes the
current CUDA stream; every step of the computation runs in the library's kernels.
PyTorch provides device memory, streams and process groups only.

Layer semantics (P:n = PAPER.md, S:n = SPEC.md lines):
  conv_forward / conv_backward_data / conv_backward_weight
  relu_*  S:196-213   pool_*  S:160-177   lrn_*  S:214-231   ip_*  S:178-195
  softmax_loss  S:250-267   sgd_update
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence, Tuple, Union

from . import _abi
from ._abi import (CAFFE_BF16, CAFFE_F32, CAFFE_I32, CAFFE_MATH_BF16, CAFFE_MATH_FP32, CAFFE_MATH_TF32,
                   CaffeError, call, load)

__all__ = ["load", "CaffeError", "conv_forward", "conv_backward_data", "conv_backward_weight", "conv_output_shape",
           "relu_forward", "relu_backward", "pool_forward", "pool_backward", "pool_output_shape", "lrn_forward",
           "lrn_backward", "ip_forward", "ip_backward_data", "ip_backward_weight", "im2col", "col2im",
           "softmax_loss", "sgd_update", "MATH"]

MATH = {"fp32": CAFFE_MATH_FP32, "tf32": CAFFE_MATH_TF32, "bf16": CAFFE_MATH_BF16}

_torch = None


def _t():
    global _torch
    if _torch is None:
        import torch
        _torch = torch
    return _torch


def _pair(v) -> Tuple[int, int]:
    return (int(v), int(v)) if isinstance(v, int) else (int(v[0]), int(v[1]))


def _dtype_code(t) -> int:
    torch = _t()
    if t.dtype == torch.float32:
        return CAFFE_F32
    if t.dtype == torch.bfloat16:
        return CAFFE_BF16
    if t.dtype == torch.int32:
        return CAFFE_I32
    if t.dtype == torch.uint8:
        return _abi.CAFFE_U8
    if t.dtype == torch.int8:
        return _abi.CAFFE_I8
    raise TypeError(f"unsupported dtype {t.dtype}")


def _shape4(shape) -> Tuple[int, int, int, int]:
    s = tuple(int(x) for x in shape)
    if len(s) == 4:
        return s
    if len(s) == 2:
        return (s[0], s[1], 1, 1)
    if len(s) == 1:
        return (1, s[0], 1, 1)
    raise ValueError(f"blob shape must have 1, 2 or 4 axes, got {s}")


def layout_of(t) -> int:
    """CAFFE_NHWC for a 4-D torch.channels_last tensor, CAFFE_NCHW for a contiguous one."""
    torch = _t()
    if t.dim() == 4 and t.is_contiguous(memory_format=torch.channels_last) and not t.is_contiguous():
        return _abi.CAFFE_NHWC
    if t.is_contiguous():
        return _abi.CAFFE_NCHW
    raise ValueError("caffe_b200 blobs must be contiguous (NCHW) or channels_last (NHWC)")


def blob(t, shape=None, host_ok=False) -> _abi.Blob:
    """Describe a CUDA tensor as a caffe_blob: contiguous -> NCHW, channels_last -> NHWC.  With
    host_ok=True a pinned host tensor is accepted too (the kernels read it through unified addressing
    over PCIe) -- only for read-only inputs such as an image batch handed to conv_pack_bottom."""
    if t is None:
        return None
    if not t.is_cuda and not (host_ok and t.is_pinned()):
        raise ValueError("caffe_b200 blobs must live on a CUDA device" +
                         (" (or in pinned host memory)" if host_ok else ""))
    lay = layout_of(t)
    n, c, h, w = _shape4(t.shape if shape is None else shape)
    return _abi.Blob(ctypes.c_void_p(t.data_ptr()), _abi.Shape4(n, c, h, w), _dtype_code(t), lay)


def empty_like_layout(shape, dtype, device, like=None, nhwc=None):
    """Allocate a 4-D blob in the layout of `like` (or NHWC if nhwc=True)."""
    torch = _t()
    if nhwc is None:
        nhwc = like is not None and layout_of(like) == _abi.CAFFE_NHWC
    if nhwc and len(shape) == 4:
        return torch.empty(tuple(shape), dtype=dtype, device=device, memory_format=torch.channels_last)
    return torch.empty(tuple(shape), dtype=dtype, device=device)


def _bp(b):
    return ctypes.byref(b) if b is not None else None


def _stream():
    return ctypes.c_void_p(_t().cuda.current_stream().cuda_stream)


# ------------------------------------------------------------------ workspace (caller-owned device memory)
_ws = {}
_ws_retired = []


def workspace(nbytes: int, device=None):
    """Return (ptr, size) of a 1024-byte-aligned scratch buffer of >= nbytes on `device` (cached, grows)."""
    torch = _t()
    if nbytes == 0:
        return None, 0
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    buf = _ws.get(dev)
    if buf is None or buf.numel() < nbytes + 1024:
        if buf is not None:
            # a CUDA graph captured earlier may still replay kernels on the old buffer: keep it alive
            _ws_retired.append(buf)
        buf = torch.empty(int(nbytes * 1.1) + 2048, dtype=torch.uint8, device=dev)
        _ws[dev] = buf
    p = buf.data_ptr()
    off = (-p) % 1024
    return ctypes.c_void_p(p + off), buf.numel() - off


def _conv_desc(kernel, stride, pad, group, math, relu=False, prepacked=False, wprepacked=False):
    kh, kw = _pair(kernel)
    sh, sw = _pair(stride)
    ph, pw = _pair(pad)
    flags = ((_abi.CAFFE_FUSE_RELU if relu else 0) | (_abi.CAFFE_BOTTOM_PREPACKED if prepacked else 0) |
             (_abi.CAFFE_WEIGHTS_PREPACKED if wprepacked else 0))
    return _abi.ConvDesc(kh, kw, sh, sw, ph, pw, int(group), MATH[math] if isinstance(math, str) else int(math), flags)


def _ws_arg(ws):
    """(ptr, bytes) of a caller-owned workspace tensor (1 KB aligned start)."""
    p = ws.data_ptr()
    off = (-p) % 1024
    return ctypes.c_void_p(p + off), ws.numel() * ws.element_size() - off


def conv_bottom_workspace(x_shape, w_shape, stride=1, pad=0, group=1, math="bf16", device=None):
    """A dedicated workspace tensor for conv_pack_bottom + conv_forward/conv_backward_weight with
    prepacked=True on one layer (the larger of the two passes' sizes)."""
    torch = _t()
    kh, kw = w_shape[2], w_shape[3]
    d = _conv_desc((kh, kw), stride, pad, group, math)
    n = 0
    for pass_ in (_abi.CAFFE_PASS_FORWARD, _abi.CAFFE_PASS_BACKWARD_WEIGHT):
        v = ctypes.c_size_t()
        call("caffe_conv_workspace_size", ctypes.byref(d), _abi.Shape4(*_shape4(x_shape)),
             _abi.Shape4(*_shape4(w_shape)), int(pass_), ctypes.byref(v))
        n = max(n, v.value)
    return torch.empty(n + 2048, dtype=torch.uint8, device=device or torch.device("cuda"))


def conv_pack_bottom(x, w, stride=1, pad=0, group=1, math="bf16", ws=None):
    """Build the tensor-core operand of x once into `ws` (caffe_conv_pack_bottom) for later
    conv_forward / conv_backward_weight calls with prepacked=True and the same ws."""
    kh, kw = w.shape[2], w.shape[3]
    d = _conv_desc((kh, kw), stride, pad, group, math)
    p, n = _ws_arg(ws)
    bx, bw = blob(x, host_ok=True), blob(w)
    call("caffe_conv_pack_bottom", ctypes.byref(d), ctypes.byref(bx), ctypes.byref(bw), p, n, _stream())


def conv_output_shape(in_shape, num_output, kernel, stride=1, pad=0, group=1):
    d = _conv_desc(kernel, stride, pad, group, "fp32")
    out = _abi.Shape4()
    call("caffe_conv_output_shape", ctypes.byref(d), _abi.Shape4(*_shape4(in_shape)), int(num_output), ctypes.byref(out))
    return (out.n, out.c, out.h, out.w)


def _conv_ws(d, in_shape, w_shape, pass_):
    n = ctypes.c_size_t()
    call("caffe_conv_workspace_size", ctypes.byref(d), _abi.Shape4(*_shape4(in_shape)), _abi.Shape4(*_shape4(w_shape)),
         int(pass_), ctypes.byref(n))
    return workspace(n.value)


def conv_pack_weights(w, in_shape, stride=1, pad=0, group=1, math="bf16", pass_=0, ws=None):
    """Write the weight operand of pass_ (0 forward, 1 data gradient) into the caller workspace `ws`
    for later calls with wprepacked=True (caffe_conv_pack_weights)."""
    kh, kw = w.shape[2], w.shape[3]
    d = _conv_desc((kh, kw), stride, pad, group, math)
    p, n = _ws_arg(ws)
    bw = blob(w)
    call("caffe_conv_pack_weights", ctypes.byref(d), _abi.Shape4(*_shape4(in_shape)), ctypes.byref(bw), int(pass_), p,
         n, _stream())


def conv_workspace(in_shape, w_shape, stride=1, pad=0, group=1, math="bf16", pass_=0, device=None):
    """A dedicated workspace tensor for one conv pass (caffe_conv_workspace_size)."""
    torch = _t()
    d = _conv_desc((w_shape[2], w_shape[3]), stride, pad, group, math)
    v = ctypes.c_size_t()
    call("caffe_conv_workspace_size", ctypes.byref(d), _abi.Shape4(*_shape4(in_shape)), _abi.Shape4(*_shape4(w_shape)),
         int(pass_), ctypes.byref(v))
    return torch.empty(v.value + 2048, dtype=torch.uint8, device=device or torch.device("cuda"))


def conv_forward(x, w, b=None, stride=1, pad=0, group=1, math="bf16", relu=False, out=None, out_dtype=None,
                 ws=None, prepacked=False, wprepacked=False):
    """Y = W (*) X + b with groups/stride/zero-pad; optional fused ReLU.  `ws` (+ prepacked)
    selects a caller workspace already holding conv_pack_bottom's operand (+ wprepacked: and
    conv_pack_weights' forward weight operand)."""
    torch = _t()
    kh, kw = w.shape[2], w.shape[3]
    d = _conv_desc((kh, kw), stride, pad, group, math, relu, prepacked, wprepacked)
    oshape = conv_output_shape(x.shape, w.shape[0], (kh, kw), stride, pad, group)
    if out is None:
        out = empty_like_layout(oshape, out_dtype or x.dtype, x.device, like=x)
    ws, wsz = _ws_arg(ws) if ws is not None else _conv_ws(d, x.shape, w.shape, _abi.CAFFE_PASS_FORWARD)
    bx, bw, bb, by = blob(x), blob(w), blob(b), blob(out)
    call("caffe_conv_forward", ctypes.byref(d), ctypes.byref(bx), ctypes.byref(bw), _bp(bb), ctypes.byref(by), ws, wsz,
         _stream())
    return out


def conv_backward_data(dy, w, in_shape, stride=1, pad=0, group=1, math="bf16", beta=0.0, out=None, out_dtype=None,
                       ws=None, wprepacked=False):
    """dX = beta*dX + W^T (*) dY."""
    torch = _t()
    kh, kw = w.shape[2], w.shape[3]
    d = _conv_desc((kh, kw), stride, pad, group, math, wprepacked=wprepacked)
    if out is None:
        out = empty_like_layout(in_shape, out_dtype or dy.dtype, dy.device, like=dy)
        out.zero_()
    ws, wsz = _ws_arg(ws) if ws is not None else _conv_ws(d, in_shape, w.shape, _abi.CAFFE_PASS_BACKWARD_DATA)
    bdy, bw, bdx = blob(dy), blob(w), blob(out)
    call("caffe_conv_backward_data", ctypes.byref(d), ctypes.byref(bdy), ctypes.byref(bw), ctypes.byref(bdx),
         float(beta), ws, wsz, _stream())
    return out


def conv_backward_data_relu(dy, w, relu_top, stride=1, pad=0, group=1, math="bf16", out=None, ws=None,
                            wprepacked=False):
    """dX = [relu_top > 0] * (W^T (*) dY): the data gradient through the ReLU whose output is this
    layer's bottom (S:154 with S:208 folded in)."""
    kh, kw = w.shape[2], w.shape[3]
    d = _conv_desc((kh, kw), stride, pad, group, math, wprepacked=wprepacked)
    if out is None:
        out = empty_like_layout(tuple(relu_top.shape), relu_top.dtype, dy.device, like=relu_top)
    ws, wsz = (_ws_arg(ws) if ws is not None
               else _conv_ws(d, tuple(relu_top.shape), w.shape, _abi.CAFFE_PASS_BACKWARD_DATA))
    bdy, bw, br, bdx = blob(dy), blob(w), blob(relu_top), blob(out)
    call("caffe_conv_backward_data_relu", ctypes.byref(d), ctypes.byref(bdy), ctypes.byref(bw), ctypes.byref(br),
         ctypes.byref(bdx), ws, wsz, _stream())
    return out


def conv_backward_weight(x, dy, w_shape, stride=1, pad=0, group=1, math="bf16", beta=0.0, dw=None, db=None,
                         bias=True, ws=None, prepacked=False):
    """dW = beta*dW + dY (*) X, db = beta*db + sum dY.  Returns (dW, db)."""
    torch = _t()
    kh, kw = w_shape[2], w_shape[3]
    d = _conv_desc((kh, kw), stride, pad, group, math, prepacked=prepacked)
    if dw is None:
        dw = torch.zeros(tuple(w_shape), dtype=torch.float32, device=x.device)
    if bias and db is None:
        db = torch.zeros((w_shape[0],), dtype=torch.float32, device=x.device)
    ws, wsz = _ws_arg(ws) if ws is not None else _conv_ws(d, x.shape, w_shape, _abi.CAFFE_PASS_BACKWARD_WEIGHT)
    bx, bdy, bdw, bdb = blob(x), blob(dy), blob(dw), blob(db) if bias else None
    call("caffe_conv_backward_weight", ctypes.byref(d), ctypes.byref(bx), ctypes.byref(bdy), ctypes.byref(bdw),
         _bp(bdb), float(beta), ws, wsz, _stream())
    return dw, (db if bias else None)


# ------------------------------------------------------------------ ReLU
def relu_forward(x, out=None, inplace=False):
    torch = _t()
    if inplace:
        out = x
    elif out is None:
        out = torch.empty_like(x)
    bx, by = blob(x), blob(out)
    call("caffe_relu_forward", ctypes.byref(bx), ctypes.byref(by), _stream())
    return out


def relu_backward(x, dy, out=None, inplace=False):
    torch = _t()
    if inplace:
        out = dy
    elif out is None:
        out = torch.empty_like(dy)
    bx, bdy, bdx = blob(x), blob(dy), blob(out)
    call("caffe_relu_backward", ctypes.byref(bx), ctypes.byref(bdy), ctypes.byref(bdx), _stream())
    return out


# ------------------------------------------------------------------ pooling
def _pool_desc(method, kernel, stride, pad):
    kh, kw = _pair(kernel)
    sh, sw = _pair(stride)
    ph, pw = _pair(pad)
    m = {"max": _abi.CAFFE_POOL_MAX, "ave": _abi.CAFFE_POOL_AVE}[method] if isinstance(method, str) else int(method)
    return _abi.PoolDesc(m, kh, kw, sh, sw, ph, pw)


def pool_output_shape(in_shape, method, kernel, stride, pad=0):
    d = _pool_desc(method, kernel, stride, pad)
    out = _abi.Shape4()
    call("caffe_pool_output_shape", ctypes.byref(d), _abi.Shape4(*_shape4(in_shape)), ctypes.byref(out))
    return (out.n, out.c, out.h, out.w)


def pool_forward(x, method, kernel, stride, pad=0, out=None, mask=None, want_mask=True, mask_dtype=None):
    """MAX/AVE pooling.  The MAX argmax mask is int32 h*W+w (Caffe) or, with mask_dtype=torch.uint8
    (or a uint8 `mask`), the window-local index -- a quarter of the bytes for the backward pass."""
    torch = _t()
    d = _pool_desc(method, kernel, stride, pad)
    oshape = pool_output_shape(x.shape, method, kernel, stride, pad)
    if out is None:
        out = empty_like_layout(oshape, x.dtype, x.device, like=x)
    if d.method == _abi.CAFFE_POOL_MAX and want_mask and mask is None:
        mask = empty_like_layout(oshape, mask_dtype or torch.int32, x.device, like=out)
    bx, by, bm = blob(x), blob(out), blob(mask) if d.method == _abi.CAFFE_POOL_MAX else None
    call("caffe_pool_forward", ctypes.byref(d), ctypes.byref(bx), ctypes.byref(by), _bp(bm), _stream())
    return out, (mask if d.method == _abi.CAFFE_POOL_MAX else None)


def pool_backward(dy, mask, in_shape, method, kernel, stride, pad=0, out=None):
    torch = _t()
    d = _pool_desc(method, kernel, stride, pad)
    if out is None:
        out = empty_like_layout(in_shape, dy.dtype, dy.device, like=dy)
    bdy, bm, bdx = blob(dy), blob(mask), blob(out)
    call("caffe_pool_backward", ctypes.byref(d), ctypes.byref(bdy), _bp(bm), ctypes.byref(bdx), _stream())
    return out


def pool_relu_backward(top, dy, mask, in_shape, kernel, stride, pad=0, out=None):
    """MAX-pool backward fused with the backward of the ReLU feeding the pool (caffe_pool_relu_backward):
    equals relu_backward(bottom, pool_backward(dy)) bit for bit; `top` is the pool forward output."""
    d = _pool_desc("max", kernel, stride, pad)
    if out is None:
        out = empty_like_layout(in_shape, dy.dtype, dy.device, like=dy)
    bt, bdy, bm, bdx = blob(top), blob(dy), blob(mask), blob(out)
    call("caffe_pool_relu_backward", ctypes.byref(d), ctypes.byref(bt), ctypes.byref(bdy), ctypes.byref(bm),
         ctypes.byref(bdx), _stream())
    return out


# ------------------------------------------------------------------ LRN
def lrn_forward(x, local_size=5, alpha=1e-4, beta=0.75, k=1.0, out=None, scale=None, want_scale=False):
    torch = _t()
    d = _abi.LrnDesc(int(local_size), float(alpha), float(beta), float(k))
    if out is None:
        out = torch.empty_like(x)
    if want_scale and scale is None:
        scale = empty_like_layout(x.shape, torch.float32, x.device, like=x)
    bx, by, bs = blob(x), blob(out), blob(scale)
    call("caffe_lrn_forward", ctypes.byref(d), ctypes.byref(bx), ctypes.byref(by), _bp(bs), _stream())
    return (out, scale) if want_scale else out


def lrn_backward(x, y, dy, local_size=5, alpha=1e-4, beta=0.75, k=1.0, scale=None, out=None):
    torch = _t()
    d = _abi.LrnDesc(int(local_size), float(alpha), float(beta), float(k))
    if out is None:
        out = torch.empty_like(dy)
    bx, by, bdy, bs, bdx = blob(x), blob(y), blob(dy), blob(scale), blob(out)
    call("caffe_lrn_backward", ctypes.byref(d), ctypes.byref(bx), ctypes.byref(by), ctypes.byref(bdy), _bp(bs),
         ctypes.byref(bdx), _stream())
    return out


# ------------------------------------------------------------------ fused pool + LRN (NEXT-1)
def pool_lrn_forward(x, kernel=3, stride=2, pad=0, local_size=5, alpha=1e-4, beta=0.75, k=1.0, pool_out=None, mask=None,
                     out=None):
    """maxpool (U8 mask) then LRN in one pass (caffe_pool_lrn_forward); returns (pool_out, mask, out)."""
    torch = _t()
    d = _pool_desc("max", kernel, stride, pad)
    oshape = pool_output_shape(x.shape, "max", kernel, stride, pad)
    if pool_out is None:
        pool_out = empty_like_layout(oshape, x.dtype, x.device, like=x)
    if mask is None:
        mask = empty_like_layout(oshape, torch.uint8, x.device, like=pool_out)
    if out is None:
        out = torch.empty_like(pool_out)
    ld = _abi.LrnDesc(int(local_size), float(alpha), float(beta), float(k))
    bx, bp, bm, by = blob(x), blob(pool_out), blob(mask), blob(out)
    call("caffe_pool_lrn_forward", ctypes.byref(d), ctypes.byref(ld), ctypes.byref(bx), ctypes.byref(bp),
         ctypes.byref(bm), ctypes.byref(by), _stream())
    return pool_out, mask, out


def lrn_pool_backward(pool_out, dy, mask, in_shape, kernel=3, stride=2, pad=0, local_size=5, alpha=1e-4, beta=0.75,
                      k=1.0, relu=True, out=None):
    """LRN backward then maxpool backward (+ the ReLU below when relu) in one pass (caffe_lrn_pool_backward)."""
    d = _pool_desc("max", kernel, stride, pad)
    if out is None:
        out = empty_like_layout(in_shape, dy.dtype, dy.device, like=dy)
    ld = _abi.LrnDesc(int(local_size), float(alpha), float(beta), float(k))
    bp, bdy, bm, bdx = blob(pool_out), blob(dy), blob(mask), blob(out)
    call("caffe_lrn_pool_backward", ctypes.byref(d), ctypes.byref(ld), ctypes.byref(bp), ctypes.byref(bdy),
         ctypes.byref(bm), int(bool(relu)), ctypes.byref(bdx), _stream())
    return out


# ------------------------------------------------------------------ inner product
def _ip_ws(math, in_shape, O, pass_):
    n = ctypes.c_size_t()
    call("caffe_ip_workspace_size", MATH[math], _abi.Shape4(*_shape4(in_shape)), int(O), int(pass_), ctypes.byref(n))
    return workspace(n.value)


def _wblob(w):
    # weight (O, K) or (O, K, 1, 1) -> (O, K, 1, 1)
    return blob(w, (w.shape[0], w.numel() // w.shape[0], 1, 1))


def ip_forward(x, w, b=None, math="bf16", relu=False, out=None, out_dtype=None):
    """Y = X W^T + b over X flattened to (N, C*H*W)."""
    torch = _t()
    O = w.shape[0]
    if out is None:
        out = torch.empty((x.shape[0], O), dtype=out_dtype or x.dtype, device=x.device)
    ws, wsz = _ip_ws(math, x.shape, O, 0)
    bx, bw, bb, by = blob(x), _wblob(w), blob(b), blob(out, (x.shape[0], O, 1, 1))
    call("caffe_ip_forward", MATH[math], _abi.CAFFE_FUSE_RELU if relu else 0, ctypes.byref(bx), ctypes.byref(bw),
         _bp(bb), ctypes.byref(by), ws, wsz, _stream())
    return out


def ip_backward_data(dy, w, in_shape, math="bf16", beta=0.0, out=None, out_dtype=None):
    torch = _t()
    if out is None:
        out = torch.zeros(tuple(in_shape), dtype=out_dtype or dy.dtype, device=dy.device)
    ws, wsz = _ip_ws(math, in_shape, w.shape[0], 1)
    bdy, bw, bdx = blob(dy, (dy.shape[0], w.shape[0], 1, 1)), _wblob(w), blob(out)
    call("caffe_ip_backward_data", MATH[math], ctypes.byref(bdy), ctypes.byref(bw), ctypes.byref(bdx), float(beta), ws,
         wsz, _stream())
    return out


def ip_backward_weight_sgd(x, dy, w, mom, w_bf16, lr, momentum, decay, grad_scale=1.0, db=None, ws=None):
    """Fused inner-product weight gradient + SGD update (S:190 then S:523): updates the FP32 master
    weights w and momentum mom in place, writes the BF16 copy w_bf16; db (optional) receives the
    bias gradient."""
    O = w.shape[0]
    ws, wsz = _ws_arg(ws) if ws is not None else _ip_ws("bf16", x.shape, O, 2)
    bx, bdy = blob(x), blob(dy, (dy.shape[0], O, 1, 1))
    bw, bm, bb = _wblob(w), _wblob(mom), _wblob(w_bf16)
    bdb = blob(db) if db is not None else None
    call("caffe_ip_backward_weight_sgd", ctypes.byref(bx), ctypes.byref(bdy), ctypes.byref(bw), ctypes.byref(bm),
         ctypes.byref(bb), _bp(bdb), float(lr), float(momentum), float(decay), float(grad_scale), ws, wsz, _stream())
    return w


def to_nchw(x, out=None):
    """NCHW copy of a channels-last blob (caffe_blob_to_nchw)."""
    torch = _t()
    if out is None:
        out = torch.empty(tuple(x.shape), dtype=x.dtype, device=x.device)
    bs, bd = blob(x), blob(out)
    call("caffe_blob_to_nchw", ctypes.byref(bs), ctypes.byref(bd), _stream())
    return out


def ip_backward_data_relu(dy, w, relu_top, math="bf16", out=None):
    """dX = [relu_top > 0] * (dY W): the data gradient through the ReLU whose output is this layer's
    bottom (S:190 with S:208 folded in)."""
    torch = _t()
    if out is None:
        out = torch.empty_like(relu_top)
    ws, wsz = _ip_ws(math, tuple(relu_top.shape), w.shape[0], 1)
    bdy, bw, br, bdx = blob(dy, (dy.shape[0], w.shape[0], 1, 1)), _wblob(w), blob(relu_top), blob(out)
    call("caffe_ip_backward_data_relu", MATH[math], ctypes.byref(bdy), ctypes.byref(bw), ctypes.byref(br),
         ctypes.byref(bdx), ws, wsz, _stream())
    return out


def ip_backward_weight(x, dy, w_shape, math="bf16", beta=0.0, dw=None, db=None, bias=True, ws=None):
    torch = _t()
    O = w_shape[0]
    if dw is None:
        dw = torch.zeros(tuple(w_shape), dtype=torch.float32, device=x.device)
    if bias and db is None:
        db = torch.zeros((O,), dtype=torch.float32, device=x.device)
    ws, wsz = _ws_arg(ws) if ws is not None else _ip_ws(math, x.shape, O, 2)
    bx, bdy, bdw = blob(x), blob(dy, (dy.shape[0], O, 1, 1)), _wblob(dw)
    bdb = blob(db) if bias else None
    call("caffe_ip_backward_weight", MATH[math], ctypes.byref(bx), ctypes.byref(bdy), ctypes.byref(bdw), _bp(bdb),
         float(beta), ws, wsz, _stream())
    return dw, (db if bias else None)


# ------------------------------------------------------------------ im2col / col2im (test entry points)
def im2col(x, n, kernel, stride=1, pad=0):
    torch = _t()
    d = _conv_desc(kernel, stride, pad, 1, "fp32")
    C = x.shape[1]
    _, _, OH, OW = conv_output_shape(x.shape, 1, kernel, stride, pad)
    kh, kw = _pair(kernel)
    col = torch.empty((C * kh * kw, OH * OW), dtype=torch.float32, device=x.device)
    bx, bc = blob(x), blob(col, (1, 1, C * kh * kw, OH * OW))
    call("caffe_im2col", ctypes.byref(d), ctypes.byref(bx), int(n), ctypes.byref(bc), _stream())
    return col


def col2im(col, in_shape, n, kernel, stride=1, pad=0, out=None):
    torch = _t()
    d = _conv_desc(kernel, stride, pad, 1, "fp32")
    if out is None:
        out = torch.zeros(tuple(in_shape), dtype=torch.float32, device=col.device)
    bc, bx = blob(col, (1, 1, col.shape[0], col.shape[1])), blob(out)
    call("caffe_col2im", ctypes.byref(d), ctypes.byref(bc), int(n), ctypes.byref(bx), _stream())
    return out


# ------------------------------------------------------------------ loss / solver glue
def softmax_loss(scores, labels, loss=None, diff=None, want_diff=True):
    torch = _t()
    if (labels.dtype != torch.int32 or not labels.is_cuda or not labels.is_contiguous()
            or labels.numel() != scores.shape[0]):
        raise ValueError("softmax_loss: labels must be a contiguous int32 CUDA tensor with one label per row "
                         f"(got {labels.dtype}, {labels.device}, {labels.numel()} labels for {scores.shape[0]} rows)")
    if loss is None:
        loss = torch.empty((), dtype=torch.float32, device=scores.device)
    if want_diff and diff is None:
        diff = torch.empty_like(scores)
    bs, bd = blob(scores, (scores.shape[0], scores.numel() // scores.shape[0], 1, 1)), \
        (blob(diff, (scores.shape[0], scores.numel() // scores.shape[0], 1, 1)) if want_diff else None)
    call("caffe_softmax_loss", ctypes.byref(bs), ctypes.c_void_p(labels.data_ptr()), ctypes.c_void_p(loss.data_ptr()),
         _bp(bd), _stream())
    return loss, diff


def sgd_update(w, g, v, lr, momentum=0.0, decay=0.0, grad_scale=1.0, w_bf16=None):
    call("caffe_sgd_update", ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(v.data_ptr()),
         ctypes.c_void_p(w_bf16.data_ptr()) if w_bf16 is not None else None, int(w.numel()), float(lr),
         float(momentum), float(decay), float(grad_scale), _stream())
    return w


# ------------------------------------------------------------------ the rest of the layer catalogue
def sigmoid_forward(x, out=None, inplace=False):
    """S:199 logistic: 1/(1+e^-x) (caffe_sigmoid_forward; in place allowed)."""
    torch = _t()
    if inplace:
        out = x
    elif out is None:
        out = torch.empty_like(x)
    bx, by = blob(x), blob(out)
    call("caffe_sigmoid_forward", ctypes.byref(bx), ctypes.byref(by), _stream())
    return out


def sigmoid_backward(y, dy, out=None, inplace=False):
    """dy * y * (1 - y) from the forward output y (caffe_sigmoid_backward)."""
    torch = _t()
    if inplace:
        out = dy
    elif out is None:
        out = torch.empty_like(dy)
    by, bdy, bdx = blob(y), blob(dy), blob(out)
    call("caffe_sigmoid_backward", ctypes.byref(by), ctypes.byref(bdy), ctypes.byref(bdx), _stream())
    return out


ELTWISE = {"prod": _abi.CAFFE_ELTWISE_PROD, "sum": _abi.CAFFE_ELTWISE_SUM, "max": _abi.CAFFE_ELTWISE_MAX}


def _blob_array(ts):
    arr = (_abi.Blob * len(ts))(*[blob(t) for t in ts])
    return arr


def _coeff_array(coeffs):
    if coeffs is None:
        return None
    return (ctypes.c_float * len(coeffs))(*[float(c) for c in coeffs])


def eltwise_forward(inputs, op="sum", coeffs=None, out=None):
    """S:235 element-wise sum (coefficients) / prod / max of >= 2 same-shaped blobs."""
    torch = _t()
    if out is None:
        out = torch.empty_like(inputs[0])
    arr = _blob_array(inputs)
    ptrs = (ctypes.POINTER(_abi.Blob) * len(inputs))(*[ctypes.pointer(arr[i]) for i in range(len(inputs))])
    bo = blob(out)
    call("caffe_eltwise_forward", int(ELTWISE[op]), len(inputs), ptrs, _coeff_array(coeffs), ctypes.byref(bo),
         _stream())
    return out


def eltwise_backward(inputs, dy, op="sum", coeffs=None, outs=None):
    """S:244 diffs of every input (list of tensors, overwritten)."""
    torch = _t()
    n = len(inputs)
    if outs is None:
        outs = [torch.empty_like(dy) for _ in range(n)]
    arr = _blob_array(inputs)
    ptrs = (ctypes.POINTER(_abi.Blob) * n)(*[ctypes.pointer(arr[i]) for i in range(n)])
    oarr = _blob_array(outs)
    optrs = (ctypes.POINTER(_abi.Blob) * n)(*[ctypes.pointer(oarr[i]) for i in range(n)])
    bdy = blob(dy)
    call("caffe_eltwise_backward", int(ELTWISE[op]), n, ptrs, _coeff_array(coeffs), ctypes.byref(bdy), optrs,
         _stream())
    return outs


def hinge_loss(scores, labels, loss=None, diff=None, want_diff=True):
    """S:271 one-vs-all L1 hinge loss and its gradient (caffe_hinge_loss)."""
    torch = _t()
    if (labels.dtype != torch.int32 or not labels.is_cuda or not labels.is_contiguous()
            or labels.numel() != scores.shape[0]):
        raise ValueError("hinge_loss: labels must be a contiguous int32 CUDA tensor with one label per row")
    if loss is None:
        loss = torch.empty((), dtype=torch.float32, device=scores.device)
    if want_diff and diff is None:
        diff = torch.empty_like(scores)
    shp = (scores.shape[0], scores.numel() // scores.shape[0], 1, 1)
    bs, bd = blob(scores, shp), (blob(diff, shp) if want_diff else None)
    call("caffe_hinge_loss", ctypes.byref(bs), ctypes.c_void_p(labels.data_ptr()), ctypes.c_void_p(loss.data_ptr()),
         _bp(bd), _stream())
    return loss, diff
