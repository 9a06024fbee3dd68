"""Pins of the catalogue-layer and solver oracles against what the paper's
spec and mathematics fix, independently of the oracle's own code (-m "not gpu"):

* SPEC worked examples (tests/golden/spec_examples.json, each with its S:n line);
* closed forms and identities (sigmoid symmetry S:204, the hinge with every margin met or with
  margins scaled, step-decay boundaries);
* library routines computing the same definition a different way: torch fp64 autograd
  (sigmoid, eltwise sum/prod/max on tie-free inputs), scikit-learn's binary hinge loss;
* central finite differences ("gradient soundness": step 1e-3, away from kinks);
* the divergence guard leaves the parameters untouched.
"""
import json
import os

import numpy as np
import pytest

import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _fd(f, x, h=1e-3):
    g = np.zeros_like(x)
    it = np.nditer(x, flags=["multi_index"])
    for _ in it:
        i = it.multi_index
        xp, xm = x.copy(), x.copy()
        xp[i] += h
        xm[i] -= h
        g[i] = (f(xp) - f(xm)) / (2 * h)
    return g


# ------------------------------------------------------------------ sigmoid
def test_sigmoid_spec_examples(oracle):
    e = GOLD["sigmoid_zero"]
    np.testing.assert_array_equal(oracle.sigmoid_forward(np.array(e["X"])), e["Y"])
    e = GOLD["sigmoid_bwd_zero"]
    y = oracle.sigmoid_forward(np.array(e["X"]))
    np.testing.assert_array_equal(oracle.sigmoid_backward(y, np.array(e["dY"])), e["dX"])


def test_sigmoid_symmetry_and_torch(oracle):
    import torch
    x = np.array([-3.0, -1.0, 1.0, 3.0])
    np.testing.assert_allclose(oracle.sigmoid_forward(x) + oracle.sigmoid_forward(-x), 1.0, rtol=0, atol=1e-15)
    X = synth.uniform((3, 4, 5, 6), 1, synth.S_X).astype(np.float64) * 6
    dY = synth.uniform(X.shape, 1, synth.S_DY).astype(np.float64)
    xt = torch.from_numpy(X).requires_grad_()
    yt = torch.sigmoid(xt)
    yt.backward(torch.from_numpy(dY))
    Y = oracle.sigmoid_forward(X)
    np.testing.assert_allclose(Y, yt.detach().numpy(), rtol=1e-14)
    np.testing.assert_allclose(oracle.sigmoid_backward(Y, dY), xt.grad.numpy(), rtol=1e-12, atol=1e-15)


def test_sigmoid_finite_differences(oracle):
    X = synth.uniform((2, 3, 4), 2, synth.S_X).astype(np.float64) * 4
    dY = synth.uniform(X.shape, 2, synth.S_DY).astype(np.float64)
    g = _fd(lambda x: float((oracle.sigmoid_forward(x) * dY).sum()), X)
    got = oracle.sigmoid_backward(oracle.sigmoid_forward(X), dY)
    assert np.abs(got - g).max() <= 1e-6 * max(1.0, np.abs(g).max())


# ------------------------------------------------------------------ eltwise
def test_eltwise_spec_examples(oracle):
    e = GOLD["eltwise_sum"]
    np.testing.assert_array_equal(oracle.eltwise_forward([np.array(v, float) for v in e["inputs"]], "sum", e["coeffs"]),
                                  e["Y"])
    e = GOLD["eltwise_max"]
    np.testing.assert_array_equal(oracle.eltwise_forward([np.array(v, float) for v in e["inputs"]], "max"), e["Y"])
    x = synth.uniform((5,), 3, synth.S_X)
    np.testing.assert_array_equal(oracle.eltwise_forward([x, x], "sum", [1, -1]), 0.0)
    for key, op in (("eltwise_sum_bwd", "sum"), ("eltwise_prod_bwd", "prod"), ("eltwise_max_tie_bwd", "max")):
        e = GOLD[key]
        d = oracle.eltwise_backward([np.array(v, float) for v in e["inputs"]], np.array(e["dY"], float), op,
                                    e.get("coeffs"))
        for a, b in zip(d, e["diffs"]):
            np.testing.assert_array_equal(a, b)


def test_eltwise_errors(oracle):
    with pytest.raises(ValueError):
        oracle.eltwise_forward([np.zeros(3)], "sum")
    with pytest.raises(ValueError):
        oracle.eltwise_forward([np.zeros(3), np.zeros(4)], "max")


@pytest.mark.parametrize("op", ["sum", "prod", "max"])
@pytest.mark.parametrize("n", [2, 3])
def test_eltwise_torch_autograd(oracle, op, n):
    import torch
    shape = (2, 3, 4, 5)
    xs = [synth.distinct_values(shape, 10 + i, spacing=0.013) + 0.0031 * i for i in range(n)]   # no ties
    coeffs = [1.5, -0.5, 2.0][:n]
    dY = synth.uniform(shape, 4, synth.S_DY).astype(np.float64)
    ts = [torch.from_numpy(x).requires_grad_() for x in xs]
    if op == "sum":
        yt = sum(c * t for c, t in zip(coeffs, ts))
    elif op == "prod":
        yt = ts[0]
        for t in ts[1:]:
            yt = yt * t
    else:
        yt = torch.stack(ts).amax(0)
    yt.backward(torch.from_numpy(dY))
    Y = oracle.eltwise_forward(xs, op, coeffs if op == "sum" else None)
    np.testing.assert_allclose(Y, yt.detach().numpy(), rtol=1e-14, atol=1e-15)
    d = oracle.eltwise_backward(xs, dY, op, coeffs if op == "sum" else None)
    for a, t in zip(d, ts):
        np.testing.assert_allclose(a, t.grad.numpy(), rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("op", ["sum", "prod", "max"])
def test_eltwise_finite_differences(oracle, op):
    shape = (2, 3, 4)
    xs = [synth.distinct_values(shape, 20 + i, spacing=0.05) + 0.011 * i for i in range(3)]
    dY = synth.uniform(shape, 5, synth.S_DY).astype(np.float64)
    coeffs = [0.5, 2.0, -1.0] if op == "sum" else None
    d = oracle.eltwise_backward(xs, dY, op, coeffs)
    for i in range(3):
        def f(x, i=i):
            ys = list(xs)
            ys[i] = x
            return float((oracle.eltwise_forward(ys, op, coeffs) * dY).sum())
        g = _fd(f, xs[i])
        assert np.abs(d[i] - g).max() <= 1e-6 * max(1.0, np.abs(g).max())


def test_eltwise_max_ties_first_wins(oracle):
    """with equal inputs the whole gradient goes to the first of them (a later input must be
    strictly greater to take it)."""
    a = np.array([1.0, 2.0, 3.0, 0.0])
    b = np.array([1.0, 5.0, 3.0, -1.0])
    c = np.array([0.0, 5.0, 3.0, 0.0])
    d = oracle.eltwise_backward([a, b, c], np.ones(4), "max")
    np.testing.assert_array_equal(d[0], [1, 0, 1, 1])
    np.testing.assert_array_equal(d[1], [0, 1, 0, 0])
    np.testing.assert_array_equal(d[2], [0, 0, 0, 0])


# ------------------------------------------------------------------ hinge loss
def test_hinge_spec_examples(oracle):
    for key in ("hinge_met", "hinge_zero"):
        e = GOLD[key]
        loss, diff = oracle.hinge_loss(np.array(e["scores"], float), e["label"])
        assert loss == e["loss"]
        np.testing.assert_array_equal(diff, e["diff"])


def test_hinge_sklearn_binary(oracle):
    """sklearn's binary hinge loss mean(max(0, 1 - y s)) over the N*K one-vs-all pairs is the same
    definition per pair: loss = K * that mean."""
    from sklearn.metrics import hinge_loss as skl
    N, K = 16, 10
    s = synth.uniform((N, K), 6, synth.S_X).astype(np.float64) * 2
    lab = synth.labels(N, K, 6)
    y = -np.ones((N, K))
    y[np.arange(N), lab] = 1
    loss, _ = oracle.hinge_loss(s, lab)
    np.testing.assert_allclose(loss, K * skl(y.ravel(), s.ravel()), rtol=1e-14)


def test_hinge_closed_forms(oracle):
    N, K = 4, 7
    lab = synth.labels(N, K, 7)
    y = -np.ones((N, K))
    y[np.arange(N), lab] = 1
    for c in (1.0, 2.5):
        loss, diff = oracle.hinge_loss(c * y, lab)
        assert loss == 0.0 and not diff.any()
    for c in (0.0, 0.25, 0.5):
        loss, diff = oracle.hinge_loss(c * y, lab)
        np.testing.assert_allclose(loss, K * (1 - c), rtol=1e-15)
        np.testing.assert_array_equal(diff, -y / N)
    with pytest.raises(ValueError):
        oracle.hinge_loss(np.zeros((2, 3)), [0, 3])


def test_hinge_finite_differences(oracle):
    N, K = 3, 5
    s = synth.distinct_values((N, K), 8, spacing=0.07)
    s = np.where(np.abs(np.abs(s) - 1.0) < 0.02, s + 0.05, s)       # away from the kinks at |s| = 1
    lab = synth.labels(N, K, 8)
    _, diff = oracle.hinge_loss(s, lab)
    g = _fd(lambda x: oracle.hinge_loss(x, lab)[0], s)
    np.testing.assert_allclose(diff, g, rtol=1e-9, atol=1e-12)


# ------------------------------------------------------------------ solver
def test_lr_policies_spec(oracle):
    from oracle import solver
    for key in ("lr_fixed", "lr_step", "lr_inv0"):
        e = GOLD[key]
        lr = solver.lr_at_iter(e["policy"], e["base_lr"], e["iter"], gamma=e.get("gamma", 0.0),
                               stepsize=e.get("stepsize", 1), power=e.get("power", 0.0))
        np.testing.assert_allclose(lr, e["lr"], rtol=1e-12)


def test_lr_policies_closed_forms(oracle):
    from oracle import solver
    # step: constant within a step, one factor gamma at each boundary
    assert solver.lr_at_iter("step", 0.1, 99, gamma=0.5, stepsize=100) == 0.1
    assert solver.lr_at_iter("step", 0.1, 100, gamma=0.5, stepsize=100) == 0.05
    # inv with gamma = power = 1 is base / (1 + iter)
    for it in (0, 1, 3, 99):
        np.testing.assert_allclose(solver.lr_at_iter("inv", 1.0, it, gamma=1.0, power=1.0), 1.0 / (1 + it), rtol=1e-15)
    # S:562 non-increasing
    for pol in ("step", "inv"):
        v = [solver.lr_at_iter(pol, 0.01, it, gamma=0.9 if pol == "step" else 1e-3, stepsize=7, power=0.75)
             for it in range(0, 2000, 13)]
        assert all(a >= b for a, b in zip(v, v[1:]))
    with pytest.raises(ValueError):
        solver.lr_at_iter("fixed", 0.01, -1)


def test_sgd_decay_only_spec(oracle):
    e = GOLD["sgd_decay_only"]
    w, v = oracle.sgd_update(np.array([e["w"]]), np.array([e["g"]]), np.array([e["v0"]]), e["lr"], e["momentum"],
                             e["decay"])
    # g' = g + decay*w = 0.01; v = -lr*g'; w moves toward 0
    np.testing.assert_allclose(v, -e["lr"] * e["g_prime"], rtol=1e-15)
    assert 0 < w[0] < e["w"]


def test_divergence_guard_leaves_params(oracle):
    """a non-finite loss aborts the step; every parameter and momentum is unchanged."""
    from oracle import net as onet, solver
    X = synth.mnist_pixels((2, 1, 28, 28), 1)
    X[0, 0, 0, 0] = np.nan
    params = onet.init_params(onet.LENET, X.shape, lambda n, s, k: synth.xavier(s, 1).astype(np.float64)
                              if k == "w" else np.zeros(s))
    moms = {k: (np.zeros_like(w), np.zeros_like(b)) for k, (w, b) in params.items()}
    before = {k: (w.copy(), b.copy()) for k, (w, b) in params.items()}
    with pytest.raises(solver.DivergenceError):
        onet.train_step(onet.LENET, X, params, moms, synth.labels(2, 10, 1))
    for k in params:
        np.testing.assert_array_equal(params[k][0], before[k][0])
        np.testing.assert_array_equal(params[k][1], before[k][1])
        assert not moms[k][0].any()
    with pytest.raises(solver.DivergenceError):
        solver.guarded_step(float("inf"), {}, {}, {}, 0.1, 0.9, 0.0)
