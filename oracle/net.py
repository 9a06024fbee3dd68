"""Oracle CaffeNet / LeNet training step -- TEST INFRASTRUCTURE ONLY (tests/, smoke(), bench.py
cpu_baseline and --impl reference).

Chains the oracle layer definitions in the order the paper's nets use them (Fig. 1
LeNet; CaffeNet = the paper's reference "AlexNet with variations", topology
from bvlc_reference_caffenet, reading R15: pool before LRN).  Its own layer table (shared with
nothing in the product package).  Forward, softmax loss, backward (S:154 etc.), SGD.
Everything is fp64 end to end (max pooling included: `maxpool_forward/backward(fp64=True)`).

Pins (tests/test_oracle_net.py): S:426 zero-parameter loss = ln K; an independent FP64 torch
autograd chain of the same topology (loss to 1e-12, every gradient to 1e-10 relative)
whole-LeNet central finite differences; mutations of the layer table (pool/LRN order, ReLU
placement) must fail the torch check; train_step's update against S:523 written out.
"""
from __future__ import annotations

import numpy as np

from . import (avepool_backward, conv_backward_data, conv_backward_weight, conv_forward, ip_backward,
               ip_forward, lrn_backward, lrn_forward, maxpool_backward, maxpool_forward, relu_backward,
               softmax_loss, sgd_update)

# (kind, name, params)
CAFFENET = [
    ("conv", "conv1", dict(O=96, k=11, s=4, p=0, g=1, relu=True)),
    ("pool", "pool1", dict(k=3, s=2)),
    ("lrn", "norm1", dict(n=5, alpha=1e-4, beta=0.75, kk=1.0)),
    ("conv", "conv2", dict(O=256, k=5, s=1, p=2, g=2, relu=True)),
    ("pool", "pool2", dict(k=3, s=2)),
    ("lrn", "norm2", dict(n=5, alpha=1e-4, beta=0.75, kk=1.0)),
    ("conv", "conv3", dict(O=384, k=3, s=1, p=1, g=1, relu=True)),
    ("conv", "conv4", dict(O=384, k=3, s=1, p=1, g=2, relu=True)),
    ("conv", "conv5", dict(O=256, k=3, s=1, p=1, g=2, relu=True)),
    ("pool", "pool5", dict(k=3, s=2)),
    ("ip", "fc6", dict(O=4096, relu=True)),
    ("ip", "fc7", dict(O=4096, relu=True)),
    ("ip", "fc8", dict(O=1000, relu=False)),
]
LENET = [
    ("conv", "conv1", dict(O=20, k=5, s=1, p=0, g=1, relu=False)),
    ("pool", "pool1", dict(k=2, s=2)),
    ("conv", "conv2", dict(O=50, k=5, s=1, p=0, g=1, relu=False)),
    ("pool", "pool2", dict(k=2, s=2)),
    ("ip", "ip1", dict(O=500, relu=True)),
    ("ip", "ip2", dict(O=10, relu=False)),
]


def forward_backward(layers, X, params, labels, quant=None, conv_only_first_dgrad=False):
    """One forward + backward pass.  params: {name: (W, b)} (fp64 arrays).  `quant(a)` (optional)
    rounds every GEMM operand (activations, weights, diffs) as the tensor-core path does (R12).
    Returns (loss, grads {name: (dW, db)}, activations list)."""
    q = quant or (lambda a: a)
    acts = [np.asarray(X, np.float64)]
    masks = {}
    for kind, name, P in layers:
        x = acts[-1]
        if kind == "conv":
            W, b = params[name]
            y = conv_forward(q(x), q(W), b, stride=(P["s"],) * 2, pad=(P["p"],) * 2, group=P["g"], relu=P["relu"])
        elif kind == "pool":
            y, masks[name] = maxpool_forward(x, (P["k"],) * 2, (P["s"],) * 2, fp64=True)
        elif kind == "lrn":
            y = lrn_forward(x, P["n"], P["alpha"], P["beta"], P["kk"])
        else:
            W, b = params[name]
            y = ip_forward(q(x), q(W), b)
            if P["relu"]:
                y = np.maximum(y, 0.0)
        acts.append(y)
    loss, d = softmax_loss(acts[-1], labels)
    grads = {}
    for li in range(len(layers) - 1, -1, -1):
        kind, name, P = layers[li]
        x, y = acts[li], acts[li + 1]
        if kind in ("conv", "ip") and P["relu"]:
            d = relu_backward(y, d)
        if kind == "conv":
            W, _ = params[name]
            dW, db = conv_backward_weight(q(x), q(d), W.shape, stride=(P["s"],) * 2, pad=(P["p"],) * 2, group=P["g"])
            if quant is not None:
                db = d.sum(axis=(0, 2, 3))   # the bias gradient is not a GEMM operand: unrounded dY
            grads[name] = (dW, db)
            if li > 0:
                d = conv_backward_data(q(d), q(W), x.shape, stride=(P["s"],) * 2, pad=(P["p"],) * 2, group=P["g"])
        elif kind == "ip":
            W, _ = params[name]
            dX, dW, db = ip_backward(q(x), q(W), q(d.reshape(d.shape[0], -1)))
            if quant is not None:
                db = d.reshape(d.shape[0], -1).sum(axis=0)
            grads[name] = (dW, db)
            d = dX.reshape(x.shape)
        elif kind == "pool":
            d = maxpool_backward(d, masks[name], x.shape, (P["k"],) * 2, (P["s"],) * 2, fp64=True)
        elif kind == "lrn":
            d = lrn_backward(x, d, P["n"], P["alpha"], P["beta"], P["kk"])
    return loss, grads, acts


def init_params(layers, in_shape, rng_w):
    """Parameter shapes for `layers`; values from the callable rng_w(name, shape, kind) -> array."""
    params = {}
    shape = tuple(in_shape)
    for kind, name, P in layers:
        N, C, H, W = shape if len(shape) == 4 else (shape[0], shape[1], 1, 1)
        if kind == "conv":
            ws = (P["O"], C // P["g"], P["k"], P["k"])
            params[name] = (rng_w(name, ws, "w"), rng_w(name, (P["O"],), "b"))
            OH = (H + 2 * P["p"] - P["k"]) // P["s"] + 1
            shape = (N, P["O"], OH, (W + 2 * P["p"] - P["k"]) // P["s"] + 1)
        elif kind == "pool":
            from . import pool_out_dim
            shape = (N, C, pool_out_dim(H, P["k"], P["s"], 0), pool_out_dim(W, P["k"], P["s"], 0))
        elif kind == "ip":
            K = int(np.prod(shape[1:]))
            params[name] = (rng_w(name, (P["O"], K), "w"), rng_w(name, (P["O"],), "b"))
            shape = (N, P["O"])
    return params


def train_step(layers, X, params, moms, labels, lr=0.01, momentum=0.9, decay=5e-4, quant=None):
    """Full SGD iteration: forward, backward, update.  Returns loss; updates in place.
    A non-finite loss raises solver.DivergenceError before any parameter changes."""
    loss, grads, _ = forward_backward(layers, X, params, labels, quant)
    if not np.isfinite(loss):
        from .solver import DivergenceError
        raise DivergenceError(f"non-finite loss {loss}")
    for name, (W, b) in params.items():
        dW, db = grads[name]
        vW, vb = moms[name]
        nW, nvW = sgd_update(W, dW, vW, lr, momentum, decay)
        nb, nvb = sgd_update(b, db, vb, lr, momentum, decay)
        W[...] = nW
        b[...] = nb
        vW[...] = nvW
        vb[...] = nvb
    return loss
