"""Pins for oracle/net.py (not gpu): the chained CaffeNet / LeNet training step.

The net oracle chains the layer oracles (each pinned in test_oracle_conv.py / test_oracle_layers.py)
in the topology of the paper's nets.  These tests pin the chaining itself -- layer order, ReLU
placement, pooling / LRN position, flattening, loss and the backward wiring -- against things other
than the oracle:

* S:426 "LeNet with zeroed parameters, any input -> loss = ln 10" (and ln 1000 for CaffeNet);
* an independent FP64 chain of library primitives (torch.nn.functional conv2d / max_pool2d
  ceil_mode / local_response_norm / linear / cross_entropy + autograd), written here from the
  CaffeNet definition (conv1 -> relu1 -> pool1 -> norm1 -> conv2(g2) -> ... -> fc8,
  reading R15) and S:416 (LeNet), at a reduced spatial size so it runs in seconds;
* S:436 / S:462: whole-net parameter gradients against central finite differences of the loss;
* mutation sanity (S:463 style): a wrong layer order or a dropped ReLU is caught by the torch check.
"""
import copy
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import synth


def _params(layers, in_shape, seed, bias_scale=0.1):
    from oracle import net as onet

    def rng_w(name, shape, kind):
        k = sum(map(ord, name))
        if kind == "w":
            return synth.xavier(shape, seed, synth.S_W, k).astype(np.float64)
        return synth.uniform(shape, seed, synth.S_B, k).astype(np.float64) * bias_scale

    return onet.init_params(layers, in_shape, rng_w)


def _torch_caffenet(x, p):
    """CaffeNet (bvlc_reference_caffenet order, R15), FP64 torch primitives."""
    def conv(x, name, stride=1, pad=0, groups=1):
        W, b = p[name]
        return F.relu(F.conv2d(x, W, b, stride=stride, padding=pad, groups=groups))

    def pool(x):
        return F.max_pool2d(x, 3, 2, ceil_mode=True)

    def norm(x):
        return F.local_response_norm(x, 5, alpha=1e-4, beta=0.75, k=1.0)

    x = norm(pool(conv(x, "conv1", stride=4)))
    x = norm(pool(conv(x, "conv2", pad=2, groups=2)))
    x = conv(x, "conv3", pad=1)
    x = conv(x, "conv4", pad=1, groups=2)
    x = pool(conv(x, "conv5", pad=1, groups=2))
    x = x.flatten(1)                                   # (c, h, w) order
    x = F.relu(F.linear(x, *p["fc6"]))
    x = F.relu(F.linear(x, *p["fc7"]))
    return F.linear(x, *p["fc8"])


def _torch_lenet(x, p):
    """LeNet (Fig. 1): conv1 -> pool1 -> conv2 -> pool2 -> ip1 -> relu -> ip2."""
    x = F.max_pool2d(F.conv2d(x, *p["conv1"]), 2, 2, ceil_mode=True)
    x = F.max_pool2d(F.conv2d(x, *p["conv2"]), 2, 2, ceil_mode=True)
    x = F.relu(F.linear(x.flatten(1), *p["ip1"]))
    return F.linear(x, *p["ip2"])


def _torch_grads(fn, X, params, labels):
    tp = {k: tuple(torch.tensor(a, dtype=torch.float64, requires_grad=True) for a in v) for k, v in params.items()}
    s = fn(torch.tensor(X, dtype=torch.float64), tp)
    loss = F.cross_entropy(s, torch.tensor(labels, dtype=torch.int64))
    loss.backward()
    return float(loss.detach()), {k: (w.grad.numpy(), b.grad.numpy()) for k, (w, b) in tp.items()}


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


# small CaffeNet input: 3x63x63 -> conv1 14 -> pool1 7 -> conv2 7 -> pool2 3 -> conv3-5 3 -> pool5 1
CAFFE_SMALL = (2, 3, 63, 63)


@pytest.mark.parametrize("which", ["lenet", "caffenet"])
def test_net_matches_torch_fp64_autograd(oracle, which):
    from oracle import net as onet
    if which == "lenet":
        layers, fn, shape, K = onet.LENET, _torch_lenet, (4, 1, 28, 28), 10
        X = synth.mnist_pixels(shape, 11).astype(np.float64)
    else:
        layers, fn, shape, K = onet.CAFFENET, _torch_caffenet, CAFFE_SMALL, 1000
        X = synth.uniform(shape, 11, synth.S_X).astype(np.float64) * 50.0
    params = _params(layers, shape, 5)
    lab = synth.labels(shape[0], K, 11)
    loss, grads, _ = onet.forward_backward(layers, X, params, lab)
    tloss, tgrads = _torch_grads(fn, X, params, lab)
    assert abs(loss - tloss) <= 1e-12 * abs(tloss), (loss, tloss)
    for name, (dW, db) in tgrads.items():
        assert _rel(grads[name][0], dW) < 1e-10, (name, "dW", _rel(grads[name][0], dW))
        assert _rel(grads[name][1], db) < 1e-10, (name, "db", _rel(grads[name][1], db))


@pytest.mark.parametrize("mutation", ["pool_lrn_swapped", "relu3_dropped", "fc8_relu_added"])
def test_torch_check_catches_wrong_topology(oracle, mutation):
    """A wrong layer order or ReLU placement in the oracle's CaffeNet table changes the loss or
    the gradients beyond the bar above (so the torch pin discriminates)."""
    from oracle import net as onet
    layers = copy.deepcopy(onet.CAFFENET)
    idx = {name: i for i, (_, name, _) in enumerate(layers)}
    if mutation == "pool_lrn_swapped":
        i = idx["pool1"]
        layers[i], layers[i + 1] = layers[i + 1], layers[i]
    elif mutation == "relu3_dropped":
        layers[idx["conv3"]][2]["relu"] = False
    else:
        layers[idx["fc8"]][2]["relu"] = True
    X = synth.uniform(CAFFE_SMALL, 11, synth.S_X).astype(np.float64) * 50.0
    params = _params(onet.CAFFENET, CAFFE_SMALL, 5)
    lab = synth.labels(CAFFE_SMALL[0], 1000, 11)
    loss, grads, _ = onet.forward_backward(layers, X, params, lab)
    tloss, tgrads = _torch_grads(_torch_caffenet, X, params, lab)
    worst = max(_rel(grads[k][0], tgrads[k][0]) for k in tgrads)
    assert abs(loss - tloss) > 1e-12 * abs(tloss) or worst > 1e-10


@pytest.mark.parametrize("which,K", [("lenet", 10), ("caffenet", 1000)])
def test_zero_parameter_net_loss_is_ln_k(oracle, which, K):
    """zeroed parameters, any input -> uniform logits -> loss = ln K (S:256 ln 10)."""
    from oracle import net as onet
    layers, shape = (onet.LENET, (3, 1, 28, 28)) if which == "lenet" else (onet.CAFFENET, CAFFE_SMALL)
    params = _params(layers, shape, 2)
    for k in params:
        params[k] = (np.zeros_like(params[k][0]), np.zeros_like(params[k][1]))
    X = synth.uniform(shape, 3, synth.S_X).astype(np.float64) * 100
    loss, grads, _ = onet.forward_backward(layers, X, params, synth.labels(shape[0], K, 3))
    assert abs(loss - math.log(K)) < 1e-14
    # zero weights: only the last layer's bias sees a gradient, (1/K - 1{label}) averaged
    last = [n for _, n, _ in layers if n in params][-1]
    np.testing.assert_allclose(grads[last][1].sum(), 0.0, atol=1e-15)


def test_lenet_finite_differences(oracle):
    """S:436 / S:462: whole-LeNet parameter gradients on a 4-sample batch vs central differences
    of the fp64 oracle loss (R19: tightened from rel 1e-2 at step 1e-3 to 1e-6 at step 1e-6)."""
    from oracle import net as onet
    shape = (4, 1, 28, 28)
    X = synth.mnist_pixels(shape, 21).astype(np.float64)
    lab = synth.labels(4, 10, 21)
    params = _params(onet.LENET, shape, 21)
    _, grads, _ = onet.forward_backward(onet.LENET, X, params, lab)
    rng = synth.gen(21, synth.S_AUX)
    h = 1e-6
    worst = 0.0
    for name in params:
        for t in range(2):                         # weight and bias
            arr = params[name][t]
            g = grads[name][t]
            scale = max(float(np.abs(g).max()), 1e-12)
            for flat in rng.choice(arr.size, size=min(6, arr.size), replace=False):
                idx = np.unravel_index(flat, arr.shape)
                old = arr[idx]
                arr[idx] = old + h
                lp, _, _ = onet.forward_backward(onet.LENET, X, params, lab)
                arr[idx] = old - h
                lm, _, _ = onet.forward_backward(onet.LENET, X, params, lab)
                arr[idx] = old
                num = (lp - lm) / (2 * h)
                worst = max(worst, abs(num - g[idx]) / scale)
    assert worst < 1e-6, worst


def test_train_step_applies_spec_sgd(oracle):
    """train_step = forward_backward + S:523 update on every parameter blob (w and b): checked
    against the update written out from the returned gradients."""
    from oracle import net as onet
    shape = (2, 1, 28, 28)
    X = synth.mnist_pixels(shape, 4).astype(np.float64)
    lab = synth.labels(2, 10, 4)
    params = _params(onet.LENET, shape, 4)
    moms = {k: (np.full_like(w, 0.01), np.full_like(b, -0.02)) for k, (w, b) in params.items()}
    before = copy.deepcopy(params)
    mom0 = copy.deepcopy(moms)
    _, grads, _ = onet.forward_backward(onet.LENET, X, before, lab)
    onet.train_step(onet.LENET, X, params, moms, lab, lr=0.1, momentum=0.9, decay=1e-3)
    for k in params:
        for t in range(2):
            v = 0.9 * mom0[k][t] - 0.1 * (grads[k][t] + 1e-3 * before[k][t])
            np.testing.assert_allclose(moms[k][t], v, rtol=0, atol=1e-15)
            np.testing.assert_allclose(params[k][t], before[k][t] + v, rtol=0, atol=1e-15)
