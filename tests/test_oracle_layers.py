"""Pins for the oracle's pooling, LRN, inner-product, ReLU, softmax-loss, SGD and
quantizer functions (not gpu)."""
import json
import math
import os

import numpy as np
import pytest

import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------------------- pooling
def test_spec_pool_examples(oracle):
    g = _load("spec_examples.json")
    for key in ("pool_max", "pool_max_s1"):
        e = g[key]
        Y, _ = oracle.maxpool_forward(np.array(e["X"]), (e["k"],) * 2, (e["s"],) * 2)
        np.testing.assert_array_equal(Y, np.array(e["Y"], np.float32), err_msg=e["cite"])
    e = g["pool_ave"]
    Y = oracle.avepool_forward(np.array(e["X"]), (e["k"],) * 2, (e["s"],) * 2)
    np.testing.assert_array_equal(Y, np.array(e["Y"]), err_msg=e["cite"])
    e = g["pool_max_bwd"]
    X = np.array(e["X"])
    _, M = oracle.maxpool_forward(X, (2, 2), (2, 2))
    dX = oracle.maxpool_backward(np.array(e["dY"]), M, X.shape, (2, 2), (2, 2))
    np.testing.assert_array_equal(dX, np.array(e["dX"], np.float32), err_msg=e["cite"])
    e = g["pool_ave_bwd"]
    dX = oracle.avepool_backward(np.array(e["dY"]), X.shape, (2, 2), (2, 2))
    np.testing.assert_array_equal(dX, np.array(e["dX"]), err_msg=e["cite"])


def test_hand_vectors_pool(oracle):
    v = _load("hand_vectors.json")
    e = v["V2_maxpool_ties"]
    Y, M = oracle.maxpool_forward(np.array(e["X"]), (3, 3), (2, 2))
    np.testing.assert_array_equal(Y, np.array(e["Y"], np.float32))
    np.testing.assert_array_equal(M, np.array(e["mask"], np.int32))
    e = v["V3_avepool_ceil_pad"]
    Y = oracle.avepool_forward(np.ones((1, 1, 4, 4)), (3, 3), (2, 2), (1, 1))
    np.testing.assert_allclose(Y, np.array(e["Y"]), rtol=1e-15)
    e = v["R5_edge"]
    assert oracle.pool_out_dim(e["H"], e["k"], e["s"], e["p"]) == e["OH"]


def test_pool_out_dims(oracle):
    assert oracle.pool_out_dim(55, 3, 2, 0) == 27
    assert oracle.pool_out_dim(27, 3, 2, 0) == 13
    assert oracle.pool_out_dim(13, 3, 2, 0) == 6
    assert oracle.pool_out_dim(24, 2, 2, 0) == 12
    assert oracle.pool_out_dim(8, 2, 2, 0) == 4
    assert oracle.pool_out_dim(6, 3, 2, 0) == 3      # ceil((6-3)/2)+1 = 3, last window clipped
    assert oracle.pool_out_dim(4, 3, 2, 1) == 3


POOL_CASES = [  # shape, k, s, p
    ((2, 3, 11, 11), (3, 3), (2, 2), (0, 0)),
    ((1, 2, 8, 8), (2, 2), (2, 2), (0, 0)),
    ((2, 2, 7, 6), (3, 3), (2, 2), (1, 1)),
    ((1, 2, 6, 9), (3, 2), (2, 3), (1, 0)),
]


@pytest.mark.parametrize("case", POOL_CASES)
def test_pool_vs_torch_fp64(oracle, case):
    torch = pytest.importorskip("torch")
    F = torch.nn.functional
    shape, k, s, p = case
    X = synth.uniform(shape, 20, synth.S_X)
    Y, M = oracle.maxpool_forward(X, k, s, p)
    yt, it = F.max_pool2d(torch.tensor(X.astype(np.float64)), k, s, p, ceil_mode=True, return_indices=True)
    np.testing.assert_array_equal(Y, yt.numpy().astype(np.float32))
    np.testing.assert_array_equal(M, it.numpy().astype(np.int32))
    xt = torch.tensor(X.astype(np.float64), requires_grad=True)
    at = F.avg_pool2d(xt, k, s, p, ceil_mode=True, count_include_pad=True)
    Ya = oracle.avepool_forward(X, k, s, p)
    np.testing.assert_allclose(Ya, at.detach().numpy(), rtol=1e-13)
    dY = synth.uniform(Ya.shape, 20, synth.S_DY).astype(np.float64)
    at.backward(torch.tensor(dY))
    np.testing.assert_allclose(oracle.avepool_backward(dY, shape, k, s, p), xt.grad.numpy(), rtol=1e-13, atol=1e-15)
    # max backward vs torch autograd (distinct values -> no ties)
    Xd = synth.distinct_values(shape, 21)
    Yd, Md = oracle.maxpool_forward(Xd, k, s, p)
    xt = torch.tensor(Xd.astype(np.float32).astype(np.float64), requires_grad=True)
    F.max_pool2d(xt, k, s, p, ceil_mode=True).backward(torch.tensor(dY))
    dX = oracle.maxpool_backward(dY, Md, shape, k, s, p)
    np.testing.assert_allclose(dX, xt.grad.numpy(), rtol=1e-6, atol=1e-6)


def test_pool_dominance_and_fd(oracle):
    """S:290 max >= ave; S:177 finite differences away from ties."""
    X = synth.uniform((2, 3, 9, 9), 22, synth.S_X)
    Ym, _ = oracle.maxpool_forward(X, (3, 3), (2, 2))
    Ya = oracle.avepool_forward(X, (3, 3), (2, 2))
    assert (Ym.astype(np.float64) >= Ya - 1e-12).all()
    Xd = synth.distinct_values((1, 2, 5, 5), 23, spacing=0.05)
    Y, M = oracle.maxpool_forward(Xd, (3, 3), (1, 1))
    dY = synth.uniform(Y.shape, 23, synth.S_DY).astype(np.float64)
    dX = oracle.maxpool_backward(dY, M, Xd.shape, (3, 3), (1, 1)).astype(np.float64)
    h = 1e-3
    for idx in np.ndindex(Xd.shape):
        a, b = Xd.copy(), Xd.copy()
        a[idx] += h
        b[idx] -= h
        num = ((oracle.maxpool_forward(a, (3, 3), (1, 1))[0].astype(np.float64) -
                oracle.maxpool_forward(b, (3, 3), (1, 1))[0]) * dY).sum() / (2 * h)
        assert abs(num - dX[idx]) < 1e-3


# ----------------------------------------------------------------------------- LRN
def test_lrn_examples(oracle):
    g = _load("spec_examples.json")["lrn_single"]
    Y = oracle.lrn_forward(np.array(g["X"]), g["n"], g["alpha"], g["beta"], g["k"])
    assert Y.ravel()[0] == pytest.approx(g["Y"][0][0][0][0], rel=1e-15)
    # alpha = 0 -> identity (k=1)
    X = synth.uniform((2, 5, 3, 3), 30, synth.S_X)
    np.testing.assert_array_equal(oracle.lrn_forward(X, 5, 0.0, 0.75, 1.0), X.astype(np.float64))
    # alpha=0, k=1, beta=1 -> bottom_diff = top_diff
    dY = synth.uniform(X.shape, 30, synth.S_DY)
    np.testing.assert_array_equal(oracle.lrn_backward(X, dY, 5, 0.0, 1.0, 1.0), dY.astype(np.float64))
    v = _load("hand_vectors.json")["V4_lrn_pixel"]
    Y = oracle.lrn_forward(np.array(v["X"], np.float64).reshape(1, 3, 1, 1), v["n"], v["alpha"], v["beta"], v["k"])
    np.testing.assert_allclose(Y.ravel(), v["Y"], rtol=1e-15)


def test_lrn_vs_torch_and_fd(oracle):
    torch = pytest.importorskip("torch")
    X = synth.uniform((2, 7, 4, 3), 31, synth.S_X).astype(np.float64) * 3
    for size, alpha, beta, k in ((5, 1e-4, 0.75, 1.0), (3, 0.5, 0.75, 2.0), (5, 2.0, 1.3, 1.0)):
        xt = torch.tensor(X, requires_grad=True)
        yt = torch.nn.functional.local_response_norm(xt, size, alpha, beta, k)
        Y = oracle.lrn_forward(X, size, alpha, beta, k)
        np.testing.assert_allclose(Y, yt.detach().numpy(), rtol=1e-13)
        dY = synth.uniform(X.shape, 31, synth.S_DY).astype(np.float64)
        yt.backward(torch.tensor(dY))
        dX = oracle.lrn_backward(X, dY, size, alpha, beta, k)
        np.testing.assert_allclose(dX, xt.grad.numpy(), rtol=1e-11, atol=1e-13)
    # FD, independent of torch
    Xs = X[:1, :, :2, :2].copy()
    dY = synth.uniform(Xs.shape, 32, synth.S_DY).astype(np.float64)
    dX = oracle.lrn_backward(Xs, dY, 3, 0.5, 0.75, 2.0)
    h = 1e-5
    for idx in np.ndindex(Xs.shape):
        a, b = Xs.copy(), Xs.copy()
        a[idx] += h
        b[idx] -= h
        num = ((oracle.lrn_forward(a, 3, 0.5, 0.75, 2.0) - oracle.lrn_forward(b, 3, 0.5, 0.75, 2.0)) * dY).sum() / (2 * h)
        assert abs(num - dX[idx]) / max(abs(num), abs(dX[idx]), 1e-8) < 1e-6


# ----------------------------------------------------------------------------- IP / ReLU / loss / SGD
def test_ip_examples_and_fd(oracle):
    g = _load("spec_examples.json")
    for key in ("ip_identity", "ip_ones_row", "ip_bias_only"):
        e = g[key]
        Y = oracle.ip_forward(np.array(e["X"]), np.array(e["W"]), np.array(e["b"]) if "b" in e else None)
        np.testing.assert_array_equal(Y, np.array(e["Y"], np.float64), err_msg=e["cite"])
    e = g["ip_bwd_outer"]
    _, dW, _ = oracle.ip_backward(np.array(e["X"]), np.array(e["W"]), np.array(e["dY"]))
    np.testing.assert_array_equal(dW, np.array(e["dW"], np.float64))
    X = synth.uniform((4, 2, 1, 5), 40, synth.S_X).astype(np.float64)
    W = synth.xavier((3, 10), 40).astype(np.float64)
    dY = synth.uniform((4, 3), 40, synth.S_DY).astype(np.float64)
    dX, dW, db = oracle.ip_backward(X, W, dY)
    h = 1e-4
    for arr, grad in ((X, dX), (W, dW)):
        for idx in np.ndindex(arr.shape):
            save = arr[idx]
            arr[idx] = save + h
            fp = (oracle.ip_forward(X, W) * dY).sum()
            arr[idx] = save - h
            fm = (oracle.ip_forward(X, W) * dY).sum()
            arr[idx] = save
            assert abs((fp - fm) / (2 * h) - grad[idx]) < 1e-9
    np.testing.assert_allclose(db, dY.sum(0), rtol=1e-15)


def test_relu_examples(oracle):
    g = _load("spec_examples.json")
    np.testing.assert_array_equal(oracle.relu_forward(np.array(g["relu_fwd"]["X"], float)), g["relu_fwd"]["Y"])
    np.testing.assert_array_equal(oracle.relu_backward(np.array(g["relu_bwd"]["X"], float),
                                                       np.array(g["relu_bwd"]["dY"], float)), g["relu_bwd"]["dX"])
    y = oracle.relu_forward(np.array([-0.0, -3.0], np.float32))
    assert not np.signbit(y).any()  # R10: +0.0 for x <= 0


def test_softmax_loss_examples(oracle):
    g = _load("spec_examples.json")
    loss, _ = oracle.softmax_loss(np.zeros((3, 10)), np.array([0, 4, 9]))
    assert loss == pytest.approx(math.log(10), abs=1e-15)
    assert loss == pytest.approx(g["softmax_uniform"]["loss"], abs=1e-6)
    e = g["softmax_peaked"]
    loss, _ = oracle.softmax_loss(np.array(e["scores"], float), np.array(e["label"]))
    assert loss == pytest.approx(e["loss"], rel=1e-4)
    e = g["softmax_diff"]
    _, d = oracle.softmax_loss(np.array(e["scores"], float), np.array(e["label"]))
    np.testing.assert_allclose(d, e["diff"], rtol=1e-15)
    s = synth.uniform((5, 7), 41, synth.S_X).astype(np.float64) * 4
    lab = synth.labels(5, 7, 41)
    loss, d = oracle.softmax_loss(s, lab)
    np.testing.assert_allclose(d.sum(1), 0, atol=1e-15)
    h = 1e-5
    for idx in np.ndindex(s.shape):
        a, b = s.copy(), s.copy()
        a[idx] += h
        b[idx] -= h
        num = (oracle.softmax_loss(a, lab)[0] - oracle.softmax_loss(b, lab)[0]) / (2 * h)
        assert abs(num - d[idx]) < 1e-9


def test_sgd_examples(oracle):
    g = _load("spec_examples.json")
    for key in ("sgd_plain", "sgd_momentum"):
        e = g[key]
        w, v = oracle.sgd_update(np.array([e["w"]]), np.array([e["g"]]), np.array([e["v0"]]),
                                 e["lr"], e["momentum"], e["decay"])
        assert v[0] == pytest.approx(e["v"], abs=1e-15) and w[0] == pytest.approx(e["w_new"], abs=1e-15)
    # S:528 decay-only pull toward 0; S:558 zero-LR fixed point
    w, v = oracle.sgd_update(np.array([1.0]), np.array([0.0]), np.array([0.0]), 0.1, 0.0, 0.01)
    assert w[0] < 1.0
    w0 = synth.uniform((8,), 42, synth.S_W).astype(np.float64)
    w, _ = oracle.sgd_update(w0, np.ones(8), np.zeros(8), 0.0, 0.9, 0.0)
    np.testing.assert_array_equal(w, w0)


def test_quantizers(oracle):
    # BF16 RNE: 1 + 2^-8 is a tie between 1 and 1+2^-7 -> even (1.0); 1 + 3*2^-8 -> 1 + 2^-6 (even)
    x = np.array([1.0 + 2.0 ** -8, 1.0 + 3 * 2.0 ** -8, 1.0 + 2.0 ** -8 + 2.0 ** -20, -2.5, 3.0], np.float32)
    np.testing.assert_array_equal(oracle.quant_bf16(x), np.array([1.0, 1.0 + 2.0 ** -6, 1.0 + 2.0 ** -7, -2.5, 3.0], np.float32))
    # TF32 keeps 10 mantissa bits
    x = np.array([1.0 + 2.0 ** -11, 1.0 + 3 * 2.0 ** -11, 1.0 + 2.0 ** -10], np.float32)
    np.testing.assert_array_equal(oracle.quant_tf32_rn(x), np.array([1.0, 1.0 + 2.0 ** -9, 1.0 + 2.0 ** -10], np.float32))
    np.testing.assert_array_equal(oracle.quant_tf32_rz(x), np.array([1.0, 1.0 + 2.0 ** -10, 1.0 + 2.0 ** -10], np.float32))
    # integers in [-128, 127] are exact in bf16 (R14)
    ints = np.arange(-128, 128, dtype=np.float32)
    np.testing.assert_array_equal(oracle.quant_bf16(ints), ints)
