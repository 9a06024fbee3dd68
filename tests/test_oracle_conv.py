"""Pins for the oracle's convolution functions (not gpu).

Every check compares the oracle with something other than itself: SPEC worked
examples, hand brute-force vectors, an independent im2col+matmul written here,
FP64 torch.nn.functional (an independent library), adjoint identities, finite
differences and the invariants S:289-S:293.
"""
import json
import os

import numpy as np
import pytest

import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_spec_conv_examples(oracle):
    g = _load("spec_examples.json")
    for key in ("conv_fwd_ones", "conv_fwd_diag", "conv_fwd_pad"):
        e = g[key]
        Y = oracle.conv_forward(np.array(e["X"]), np.array(e["W"]), None,
                                stride=(e["stride"],) * 2, pad=(e["pad"],) * 2)
        np.testing.assert_array_equal(Y, np.array(e["Y"], np.float64), err_msg=e["cite"])


def test_spec_conv_backward_examples(oracle):
    # top_diff zero -> all diffs zero
    X = synth.uniform((2, 3, 5, 5), 0, synth.S_X)
    W = synth.xavier((4, 3, 3, 3), 0)
    dY = np.zeros((2, 4, 3, 3))
    dX = oracle.conv_backward_data(dY, W, X.shape, stride=(2, 2), pad=(1, 1))
    dW, db = oracle.conv_backward_weight(X, dY, W.shape, stride=(2, 2), pad=(1, 1))
    assert not dX.any() and not dW.any() and not db.any()
    # 1x1 kernel of weight w: weight_diff = sum(top_diff * input)
    X = synth.uniform((1, 1, 2, 2), 1, synth.S_X)
    dY = synth.uniform((1, 1, 2, 2), 1, synth.S_DY)
    dW, _ = oracle.conv_backward_weight(X, dY, (1, 1, 1, 1))
    assert dW[0, 0, 0, 0] == pytest.approx(float((X.astype(np.float64) * dY).sum()), rel=1e-15)


def test_hand_vector_v1(oracle):
    v = _load("hand_vectors.json")["V1_conv_g2_s2_p1"]
    c, h, w = np.meshgrid(np.arange(2), np.arange(4), np.arange(4), indexing="ij")
    X = (16 * c + 4 * h + w + 1).astype(np.float64)[None]
    W = np.array(v["W"], np.float64)
    b = np.array(v["b"], np.float64)
    kw = dict(stride=(2, 2), pad=(1, 1), group=2)
    Y = oracle.conv_forward(X, W, b, **kw)
    np.testing.assert_array_equal(Y, np.array(v["Y"], np.float64))
    dY = np.ones_like(Y)
    dW, db = oracle.conv_backward_weight(X, dY, W.shape, **kw)
    np.testing.assert_array_equal(dW, np.array(v["dW_dY1"], np.float64))
    np.testing.assert_array_equal(db, np.array(v["db_dY1"], np.float64))
    dX = oracle.conv_backward_data(dY, W, X.shape, **kw)
    np.testing.assert_array_equal(dX, np.array(v["dX_dY1"], np.float64))
    dY = np.arange(1, 9, dtype=np.float64).reshape(Y.shape)
    Y0 = oracle.conv_forward(X, W, None, **kw)
    dX = oracle.conv_backward_data(dY, W, X.shape, **kw)
    dW, _ = oracle.conv_backward_weight(X, dY, W.shape, **kw)
    t = v["inner_dY_1to8"]
    assert (Y0 * dY).sum() == t and (X * dX).sum() == t and (W * dW).sum() == t


CASES = [  # N, C, H, W, O, k, s, p, g
    (2, 3, 7, 6, 4, (3, 3), (1, 1), (1, 1), 1),
    (2, 4, 9, 9, 6, (3, 2), (2, 1), (1, 0), 2),
    (1, 6, 11, 11, 6, (5, 5), (2, 2), (2, 2), 3),
    (3, 3, 15, 15, 4, (11, 11), (4, 4), (0, 0), 1),   # conv1-like stride 4
    (2, 2, 5, 5, 2, (1, 1), (1, 1), (0, 0), 2),       # 1x1 grouped
]


def _im2col_matmul(X, W, b, stride, pad, g):
    """Independent lowering written here (not the oracle's): patch matrix + numpy matmul."""
    N, C, H, Wd = X.shape
    O, Cg, kh, kw = W.shape
    OH = (H + 2 * pad[0] - kh) // stride[0] + 1
    OW = (Wd + 2 * pad[1] - kw) // stride[1] + 1
    Xp = np.zeros((N, C, H + 2 * pad[0], Wd + 2 * pad[1]))
    Xp[:, :, pad[0]:pad[0] + H, pad[1]:pad[1] + Wd] = X
    Y = np.zeros((N, O, OH, OW))
    Og = O // g
    for gi in range(g):
        cols = np.zeros((N, Cg, kh, kw, OH, OW))
        for i in range(kh):
            for j in range(kw):
                cols[:, :, i, j] = Xp[:, gi * Cg:(gi + 1) * Cg,
                                      i:i + stride[0] * (OH - 1) + 1:stride[0],
                                      j:j + stride[1] * (OW - 1) + 1:stride[1]]
        cols = cols.reshape(N, Cg * kh * kw, OH * OW)
        Wm = W[gi * Og:(gi + 1) * Og].reshape(Og, -1)
        Y[:, gi * Og:(gi + 1) * Og] = np.einsum("ok,nkp->nop", Wm, cols).reshape(N, Og, OH, OW)
    return Y + (b[None, :, None, None] if b is not None else 0)


@pytest.mark.parametrize("case", CASES)
def test_conv_forward_im2col_matmul_equiv(oracle, case):
    N, C, H, W, O, k, s, p, g = case
    X = synth.uniform((N, C, H, W), 3, synth.S_X).astype(np.float64)
    Wt = synth.xavier((O, C // g) + k, 3).astype(np.float64)
    b = synth.uniform((O,), 3, synth.S_B).astype(np.float64)
    Y = oracle.conv_forward(X, Wt, b, stride=s, pad=p, group=g)
    np.testing.assert_allclose(Y, _im2col_matmul(X, Wt, b, s, p, g), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("case", CASES)
def test_conv_vs_torch_fp64(oracle, case):
    torch = pytest.importorskip("torch")
    F = torch.nn.functional
    N, C, H, W, O, k, s, p, g = case
    X = synth.uniform((N, C, H, W), 4, synth.S_X).astype(np.float64)
    Wt = synth.xavier((O, C // g) + k, 4).astype(np.float64)
    b = synth.uniform((O,), 4, synth.S_B).astype(np.float64)
    xt = torch.tensor(X, requires_grad=True)
    wt = torch.tensor(Wt, requires_grad=True)
    bt = torch.tensor(b, requires_grad=True)
    yt = F.conv2d(xt, wt, bt, stride=s, padding=p, groups=g)
    Y = oracle.conv_forward(X, Wt, b, stride=s, pad=p, group=g)
    np.testing.assert_allclose(Y, yt.detach().numpy(), rtol=1e-12, atol=1e-12)
    dY = synth.uniform(Y.shape, 4, synth.S_DY).astype(np.float64)
    yt.backward(torch.tensor(dY))
    dX = oracle.conv_backward_data(dY, Wt, X.shape, stride=s, pad=p, group=g)
    dW, db = oracle.conv_backward_weight(X, dY, Wt.shape, stride=s, pad=p, group=g)
    np.testing.assert_allclose(dX, xt.grad.numpy(), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(dW, wt.grad.numpy(), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(db, bt.grad.numpy(), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("case", CASES)
def test_conv_adjoint_identities(oracle, case):
    """<conv(X),dY> = <X, dgrad(dY)> = <W, wgrad(X,dY)>;  <b,db> = sum dY * b."""
    N, C, H, W, O, k, s, p, g = case
    X = synth.uniform((N, C, H, W), 5, synth.S_X).astype(np.float64)
    Wt = synth.xavier((O, C // g) + k, 5).astype(np.float64)
    Y = oracle.conv_forward(X, Wt, None, stride=s, pad=p, group=g)
    dY = synth.uniform(Y.shape, 5, synth.S_DY).astype(np.float64)
    dX = oracle.conv_backward_data(dY, Wt, X.shape, stride=s, pad=p, group=g)
    dW, db = oracle.conv_backward_weight(X, dY, Wt.shape, stride=s, pad=p, group=g)
    a, bb, c = (Y * dY).sum(), (X * dX).sum(), (Wt * dW).sum()
    assert bb == pytest.approx(a, rel=1e-12, abs=1e-12)
    assert c == pytest.approx(a, rel=1e-12, abs=1e-12)
    np.testing.assert_allclose(db, dY.sum(axis=(0, 2, 3)), rtol=1e-13)


def test_conv_finite_differences(oracle):
    """S:159 / S:288: analytic gradients vs central differences (fp64 so tightened to 1e-6)."""
    s, p, g = (2, 2), (1, 1), 1
    X = synth.uniform((1, 2, 5, 5), 6, synth.S_X).astype(np.float64)
    Wt = synth.xavier((3, 2, 3, 3), 6).astype(np.float64)
    b = synth.uniform((3,), 6, synth.S_B).astype(np.float64)
    dY = synth.uniform((1, 3, 3, 3), 6, synth.S_DY).astype(np.float64)
    f = lambda X_, W_, b_: (oracle.conv_forward(X_, W_, b_, stride=s, pad=p, group=g) * dY).sum()
    dX = oracle.conv_backward_data(dY, Wt, X.shape, stride=s, pad=p, group=g)
    dW, db = oracle.conv_backward_weight(X, dY, Wt.shape, stride=s, pad=p, group=g)
    h = 1e-3
    for arr, grad, which in ((X, dX, 0), (Wt, dW, 1), (b, db, 2)):
        for idx in np.ndindex(arr.shape):
            args_p = [X.copy(), Wt.copy(), b.copy()]
            args_m = [X.copy(), Wt.copy(), b.copy()]
            args_p[which][idx] += h
            args_m[which][idx] -= h
            num = (f(*args_p) - f(*args_m)) / (2 * h)
            a = grad[idx]
            assert abs(a - num) / max(abs(a), abs(num), 1e-8) < 1e-6 or abs(a - num) < 1e-9


def test_conv_sign_flip_mutation_is_caught(oracle):
    """S:463 mutation sanity: a sign-flipped data gradient must fail the adjoint identity."""
    X = synth.uniform((1, 2, 5, 5), 7, synth.S_X).astype(np.float64)
    Wt = synth.xavier((3, 2, 3, 3), 7).astype(np.float64)
    Y = oracle.conv_forward(X, Wt, None, pad=(1, 1))
    dY = synth.uniform(Y.shape, 7, synth.S_DY).astype(np.float64)
    dX = -oracle.conv_backward_data(dY, Wt, X.shape, pad=(1, 1))
    assert abs((Y * dY).sum() - (X * dX).sum()) > 1e-3


def test_conv_invariants(oracle):
    """S:289 linearity, S:293 batch decomposability, S:292 2x accumulation."""
    X = synth.uniform((2, 4, 6, 6), 8, synth.S_X).astype(np.float64)
    X2 = synth.uniform((2, 4, 6, 6), 8, synth.S_X, 1).astype(np.float64)
    Wt = synth.xavier((6, 2, 3, 3), 8).astype(np.float64)
    kw = dict(stride=(1, 1), pad=(1, 1), group=2)
    Y1, Y2 = oracle.conv_forward(X, Wt, **kw), oracle.conv_forward(X2, Wt, **kw)
    np.testing.assert_allclose(oracle.conv_forward(X + X2, Wt, **kw), Y1 + Y2, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(oracle.conv_forward(3.0 * X, Wt, **kw), 3.0 * Y1, rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(oracle.conv_forward(X[1:], Wt, **kw), Y1[1:])
    dY = synth.uniform(Y1.shape, 8, synth.S_DY).astype(np.float64)
    dW1, db1 = oracle.conv_backward_weight(X, dY, Wt.shape, beta=1.0, **kw)
    dW2, db2 = oracle.conv_backward_weight(X, dY, Wt.shape, beta=1.0, dW=dW1, db=db1, **kw)
    np.testing.assert_array_equal(dW2, 2 * dW1)
    np.testing.assert_array_equal(db2, 2 * db1)
    dX1 = oracle.conv_backward_data(dY, Wt, X.shape, **kw)
    dX2 = oracle.conv_backward_data(dY, Wt, X.shape, beta=1.0, dX=dX1, **kw)
    np.testing.assert_array_equal(dX2, 2 * dX1)


def test_conv_fused_relu(oracle):
    X = synth.uniform((1, 3, 6, 6), 9, synth.S_X)
    Wt = synth.xavier((4, 3, 3, 3), 9)
    b = synth.uniform((4,), 9, synth.S_B)
    Y = oracle.conv_forward(X, Wt, b, pad=(1, 1))
    Yr = oracle.conv_forward(X, Wt, b, pad=(1, 1), relu=True)
    np.testing.assert_array_equal(Yr, np.maximum(Y, 0.0))


def test_conv_output_dim_rule(oracle):
    # S:122 floor; CaffeNet shapes
    assert oracle.conv_out_dim(227, 11, 4, 0) == 55
    assert oracle.conv_out_dim(27, 5, 1, 2) == 27
    assert oracle.conv_out_dim(13, 3, 1, 1) == 13
    assert oracle.conv_out_dim(28, 5, 1, 0) == 24
    assert oracle.conv_out_dim(8, 3, 2, 0) == 3       # floor((8-3)/2)+1
    assert oracle.conv_out_dim(2, 5, 1, 1) == -1      # kernel larger than padded input


def test_im2col_brute_force_and_adjoint(oracle):
    X = synth.int_pixels((2, 3, 6, 5), 10, lo=-8, hi=8)
    k, s, p = (3, 2), (2, 1), (1, 1)
    col = oracle.im2col(X, 1, k, s, p)
    OH, OW = (6 + 2 - 3) // 2 + 1, (5 + 2 - 2) // 1 + 1
    assert col.shape == (3 * 3 * 2, OH * OW)
    for c in range(3):
        for i in range(3):
            for j in range(2):
                for y in range(OH):
                    for x in range(OW):
                        h, w = y * 2 - 1 + i, x - 1 + j
                        want = X[1, c, h, w] if (0 <= h < 6 and 0 <= w < 5) else 0.0
                        assert col[(c * 3 + i) * 2 + j, y * OW + x] == want
    # col2im is the adjoint of im2col; on small integers every FP32 sum is exact.
    dcol = synth.int_pixels(col.shape, 11, lo=-8, hi=8)
    dX = oracle.col2im(dcol, X.shape, 1, k, s, p)
    assert float((col.astype(np.float64) * dcol).sum()) == float((X[1].astype(np.float64) * dX[1]).sum())
    assert not dX[0].any()
    # col2im of (W^T dY) equals the conv data gradient
    Wt = synth.int_pixels((4, 3, 3, 2), 12, lo=-3, hi=3)
    dY = synth.int_pixels((2, 4, OH, OW), 13, lo=-3, hi=3)
    dcol = (Wt.reshape(4, -1).T @ dY[1].reshape(4, -1)).astype(np.float32)
    dX = oracle.col2im(dcol, X.shape, 1, k, s, p)
    ref = oracle.conv_backward_data(dY, Wt, X.shape, stride=s, pad=p)
    np.testing.assert_array_equal(dX[1], ref[1].astype(np.float32))
