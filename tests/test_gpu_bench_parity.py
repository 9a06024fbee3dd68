"""Parity of the exact configuration bench.py times (-m gpu): CaffeNet, batch 256, int8 image batch,
BF16 tensor-core math, the three-stream step captured in a CUDA graph and replayed -- the same
persistent multi-unit tensor-core schedule (CTA pairs chosen automatically, 12-24 work units per
CTA pair, accumulator double buffers and barrier phases carried across units) the headline number
comes from.

Teacher-forced (every pass is checked on the GPU's OWN inputs of that pass: its stored bottom, the
top diff it consumed and the weights it read), against the oracle (Sec. 3.3:
"identical results ... with tests to prove it"):

* conv / inner-product forward and data gradient on 8 images spread over the batch (first and last
  image, so the first and the ragged last M tile of every pass), the BF16 output within 1 BF16 ulp
  of RNE(oracle) per element (reading R12 for BF16-stored outputs) and rel-L2 <= 1e-3;
* weight and bias gradients over all 256 images (FP32 outputs): rel-L2 <= 1e-3 and per element
  within 1e-3 of the largest gradient of the layer;
* max pool forward values and argmax (U8 window-local mask decoded to Caffe's h*W+w) and the
  ReLU-fused backward over the whole batch: bit-exact (readings R7, R8);
* LRN forward and backward over the whole batch: within 1 BF16 ulp of RNE(oracle) per element;
* softmax loss and its BF16 gradient; the SGD update of all 61 M parameters.
"""
import numpy as np
import pytest

import synth
from _helpers import assert_bf16_ulp, assert_tc_close, host, rel_l2


def _q(a):
    """RNE BF16 of an oracle result: the rel-L2 bar for BF16-stored outputs compares against the
    oracle rounded the way the output is stored (reading R12)."""
    import oracle
    return oracle.quant_bf16(np.asarray(a, np.float32))

pytestmark = pytest.mark.gpu

B = 256
SAMPLE = [0, 37, 73, 110, 146, 183, 219, 255]
LRN = dict(size=5, alpha=1e-4, beta=0.75, k=1.0)
LR, MOM, DECAY = 0.01, 0.9, 5e-4


@pytest.fixture(scope="module")
def stepped():
    import torch
    from paper_1408_5093_b200 import nets
    dev = torch.device("cuda")
    # exactly bench.py's construction, warm-up and captured step
    net = nets.Net(nets.CAFFENET, B, nets.CAFFENET_INPUT, dev, math="bf16", seed=0, input_i8=True)
    X = synth.int_pixels((B, 3, 227, 227), 1000)
    lab = synth.labels(B, 1000, 1000)
    net.a[0].copy_(torch.from_numpy(X).to(net.a[0].dtype))
    net.labels.copy_(torch.from_numpy(lab))
    for _ in range(3):
        net.step()
    torch.cuda.synchronize()
    net.capture(allreduce=None)
    torch.cuda.synchronize()
    snap = dict(params=net.params.clone(), mom=net.mom.clone(), wq=net.params_bf16.clone())
    net.graph.replay()
    torch.cuda.synchronize()
    # weights the step read (the step updates them in place at its end)
    W = {i: net.canonical(i, snap["wq"][net.W[i].storage_offset() - net.params.storage_offset():][:net.W[i].numel()]
                          .view(net.W[i].shape).float().cpu().numpy().astype(np.float64)) for (i, _, _) in net.pspecs}
    Bs = {i: snap["params"][net.B[i].storage_offset() - net.params.storage_offset():][:net.B[i].numel()]
          .cpu().numpy().astype(np.float64) for (i, _, _) in net.pspecs}
    return net, snap, W, Bs, lab


def _a(net, i, idx=None):
    t = net.a[i] if idx is None else net.a[i][idx]
    return host(t).astype(np.float64)


def _d(net, i, idx=None):
    n = len(net.layers)
    t = net.dscores if i == n - 1 else net.d[i]
    t = t if idx is None else t[idx]
    return host(t).astype(np.float64)


def _layer(net, name):
    return next(i for i, L in enumerate(net.layers) if L.name == name)


def _relu_below(net, i):
    """True when d[i] carries the ReLU mask of the layer below (conv/ip with ReLU)."""
    return i > 0 and net.layers[i - 1].kind in ("conv", "ip") and net.layers[i - 1].relu


def _conv_atol(ref):
    # FP32 accumulation of up to 3,456 products: admit 2^-12 of the layer's RMS output where the
    # exact value cancels to ~0 (a BF16 ulp there is smaller than the FP32 sum's own rounding)
    return float(np.sqrt(np.mean(np.square(ref)))) * 2.0 ** -12


@pytest.mark.parametrize("name", ["conv1", "conv2", "conv3", "conv4", "conv5"])
def test_conv_forward_bench_config(oracle, stepped, name):
    net, _, W, Bs, _ = stepped
    i = _layer(net, name)
    L = net.layers[i]
    x = _a(net, i, SAMPLE)
    ref = oracle.conv_forward(x, W[i], Bs[i], stride=(L.stride,) * 2, pad=(L.pad,) * 2, group=L.group, relu=L.relu)
    got = _a(net, i + 1, SAMPLE)
    assert_tc_close(got, _q(ref), f"{name} fwd rel-L2")
    assert_bf16_ulp(got, ref, f"{name} fwd", atol=_conv_atol(ref))


@pytest.mark.parametrize("name", ["conv2", "conv3", "conv4", "conv5"])
def test_conv_backward_data_bench_config(oracle, stepped, name):
    net, _, W, _, _ = stepped
    i = _layer(net, name)
    L = net.layers[i]
    dy = _d(net, i + 1, SAMPLE)
    ref = oracle.conv_backward_data(dy, W[i], (len(SAMPLE),) + tuple(net.shapes[i][1:]), stride=(L.stride,) * 2,
                                    pad=(L.pad,) * 2, group=L.group)
    if _relu_below(net, i):            # caffe_conv_backward_data_relu: the mask of relu3 / relu4
        ref = oracle.relu_backward(_a(net, i, SAMPLE), ref)
    got = _d(net, i, SAMPLE)
    assert_tc_close(got, _q(ref), f"{name} dgrad rel-L2")
    assert_bf16_ulp(got, ref, f"{name} dgrad", atol=_conv_atol(ref))


@pytest.mark.parametrize("name", ["conv1", "conv2", "conv3", "conv4", "conv5"])
def test_conv_backward_weight_bench_config(oracle, stepped, name):
    net, _, W, _, _ = stepped
    i = _layer(net, name)
    L = net.layers[i]
    x = _a(net, i)
    dy = _d(net, i + 1)
    rW, rb = oracle.conv_backward_weight(x, dy, W[i].shape, stride=(L.stride,) * 2, pad=(L.pad,) * 2, group=L.group)
    gW, gb = host(net.dW[i]).astype(np.float64), host(net.dB[i]).astype(np.float64)
    assert_tc_close(gW, rW, f"{name} dW (256 images)")
    assert_tc_close(gb, rb, f"{name} db (256 images)")
    assert np.abs(gW - rW).max() <= 1e-3 * np.abs(rW).max(), f"{name} dW worst element"
    assert np.abs(gb - rb).max() <= 1e-3 * np.abs(rb).max(), f"{name} db worst element"


@pytest.mark.parametrize("name", ["pool1", "pool2", "pool5"])
def test_maxpool_bench_config(oracle, stepped, name):
    net, _, _, _, _ = stepped
    i = _layer(net, name)
    L = net.layers[i]
    x = host(net.a[i])
    rY, rM = oracle.maxpool_forward(x, (L.kernel,) * 2, (L.stride,) * 2)
    np.testing.assert_array_equal(host(net.a[i + 1]), rY)
    loc = host(net.mask[i]).astype(np.int64)
    OH, OW = rY.shape[2:]
    py = np.arange(OH).reshape(1, 1, OH, 1)
    px = np.arange(OW).reshape(1, 1, 1, OW)
    np.testing.assert_array_equal((py * L.stride + loc // L.kernel) * x.shape[3] + (px * L.stride + loc % L.kernel),
                                  rM)
    # backward (the ReLU of the conv below folded in): FP32 gather in the R8 order, stored as RNE
    # BF16.  pool1/pool2 run fused with the LRN above (caffe_lrn_pool_backward: the LRN's bottom diff
    # is never stored), so their top diff is that LRN backward recomputed here by the separate call
    # (itself checked against the oracle in test_lrn_bench_config)
    dy = host(_pool_top_diff(net, i))
    ref = oracle.maxpool_backward(dy, rM, x.shape, (L.kernel,) * 2, (L.stride,) * 2)
    if _relu_below(net, i):
        ref = oracle.relu_backward(x, ref)
    np.testing.assert_array_equal(host(net.d[i]), oracle.quant_bf16(ref))


def _pool_top_diff(net, i):
    """The top diff pool layer i consumed: d[i+1], or -- pool fused with the LRN above -- the LRN's
    bottom diff from the separate caffe_lrn_backward on the step's own blobs."""
    import paper_1408_5093_b200 as cb
    from paper_1408_5093_b200 import nets
    if not (net._pool_lrn(i) and net.fuse_lrn_pool_backward):
        return net.d[i + 1]
    return cb.lrn_backward(net.a[i + 1], net.a[i + 2], net.d[i + 2], **nets.LRN)


@pytest.mark.parametrize("name", ["norm1", "norm2"])
def test_lrn_bench_config(oracle, stepped, name):
    net, _, _, _, _ = stepped
    i = _layer(net, name)
    x = _a(net, i)
    ref = oracle.lrn_forward(x, **LRN)
    assert_bf16_ulp(_a(net, i + 1), ref, f"{name} fwd")
    dy = _d(net, i + 1)
    ref = oracle.lrn_backward(x, dy, **LRN)
    got = host(_pool_top_diff(net, i - 1)).astype(np.float64)
    assert_tc_close(got, _q(ref), f"{name} bwd rel-L2")
    # the kernel uses the stored BF16 top in the cross-channel term (-2ab/n x sum dy y / S): admit its
    # rounding where the first term cancels
    assert_bf16_ulp(got, ref, f"{name} bwd", atol=float(np.abs(ref).max()) * 2.0 ** -16)


@pytest.mark.parametrize("name", ["fc6", "fc7", "fc8"])
def test_inner_product_bench_config(oracle, stepped, name):
    net, _, W, Bs, lab = stepped
    i = _layer(net, name)
    L = net.layers[i]
    n = len(net.layers)
    x = _a(net, i)
    ref = oracle.ip_forward(x, W[i], Bs[i])
    if L.relu:
        ref = oracle.relu_forward(ref)
    last = i + 1 == n - 1
    got = host(net.scores).astype(np.float64) if last else _a(net, i + 1).reshape(B, -1)
    assert_tc_close(got, ref if last else _q(ref), f"{name} fwd rel-L2")
    if last:   # FP32 scores
        assert np.abs(got - ref).max() <= 1e-4 * np.abs(ref).max()
    else:
        assert_bf16_ulp(got, ref, f"{name} fwd", atol=_conv_atol(ref))
    dy = _d(net, i + 1).reshape(B, -1)
    rdX, rdW, rdb = oracle.ip_backward(x, W[i], dy)
    gW, gb = net.canonical(i, host(net.dW[i])).astype(np.float64), host(net.dB[i]).astype(np.float64)
    assert_tc_close(gW, rdW, f"{name} dW")
    assert_tc_close(gb, rdb, f"{name} db")
    assert np.abs(gW - rdW).max() <= 1e-3 * np.abs(rdW).max()
    rdX = rdX.reshape((B,) + tuple(net.shapes[i][1:]))
    if _relu_below(net, i):            # caffe_ip_backward_data_relu (relu6 / relu7 mask)
        rdX = oracle.relu_backward(x.reshape(rdX.shape), rdX)
    got = _d(net, i)
    assert_tc_close(got, _q(rdX), f"{name} dgrad rel-L2")
    assert_bf16_ulp(got, rdX, f"{name} dgrad", atol=_conv_atol(rdX))


def test_softmax_loss_bench_config(oracle, stepped):
    net, _, _, _, lab = stepped
    lo, dref = oracle.softmax_loss(host(net.scores), lab)
    assert abs(float(net.loss) - lo) <= 1e-5 * (abs(lo) + 1)
    assert_bf16_ulp(host(net.dscores), dref, "softmax diff (BF16)", atol=2.0 ** -30)


def test_sgd_update_bench_config(oracle, stepped):
    """All 61 M parameters: the per-layer side-stream updates of the step (R18) against the
    oracle update of the pre-step weights with the step's gradients; BF16 copy = RNE(FP32 master)."""
    net, snap, _, _, _ = stepped
    w0, v0 = snap["params"].cpu().numpy(), snap["mom"].cpu().numpy()
    g = net.grads.cpu().numpy()
    rw, rv = oracle.sgd_update(w0, g, v0, LR, MOM, DECAY)
    w1, v1 = net.params.cpu().numpy(), net.mom.cpu().numpy()
    assert np.all(np.abs(w1 - rw) <= 1e-5 * (np.abs(rw) + 1)), np.abs(w1 - rw).max()
    assert np.all(np.abs(v1 - rv) <= 1e-5 * (np.abs(rv) + 1)), np.abs(v1 - rv).max()
    np.testing.assert_array_equal(net.params_bf16.float().cpu().numpy(), oracle.quant_bf16(w1))


def test_loss_is_finite_and_reproducible(stepped):
    """Replaying the captured step from the same state gives bit-identical gradients."""
    import torch
    net, snap, _, _, _ = stepped
    g1 = net.grads.clone()
    p1, m1, q1 = net.params.clone(), net.mom.clone(), net.params_bf16.clone()
    net.params.copy_(snap["params"])
    net.mom.copy_(snap["mom"])
    net.params_bf16.copy_(snap["wq"])
    net.graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(net.grads, g1)
    assert torch.equal(net.params, p1) and torch.equal(net.mom, m1) and torch.equal(net.params_bf16, q1)
    assert np.isfinite(float(net.loss))
