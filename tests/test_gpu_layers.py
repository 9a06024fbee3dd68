"""GPU parity of the neighbour layers (ReLU, pooling, LRN, inner product), im2col/col2im,
softmax-with-loss and the SGD update against the CPU oracle (-m gpu)."""
import numpy as np
import pytest

import synth
from _helpers import assert_bf16_ulp, assert_fp32_close, assert_tc_close, cuda, host

pytestmark = pytest.mark.gpu


def test_im2col_col2im_bit_exact(oracle):
    import paper_1408_5093_b200 as cb
    for (shape, k, s, p) in [((2, 3, 9, 8), (3, 3), (2, 1), (1, 1)), ((1, 3, 23, 23), (11, 11), (4, 4), (0, 0)),
                             ((2, 5, 7, 7), (5, 5), (1, 1), (2, 2))]:
        X = synth.uniform(shape, 1, synth.S_X)
        for n in range(shape[0]):
            col = cb.im2col(cuda(X), n, k, s, p)
            np.testing.assert_array_equal(host(col), oracle.im2col(X, n, k, s, p))
            dcol = synth.uniform(tuple(col.shape), 1, synth.S_DY, n)
            dX = cb.col2im(cuda(dcol), shape, n, k, s, p)
            ref = oracle.col2im(dcol, shape, n, k, s, p)
            np.testing.assert_array_equal(host(dX)[n], ref[n])


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_relu(oracle, dtype):
    import torch
    import paper_1408_5093_b200 as cb
    X = synth.uniform((3, 5, 7, 9), 2, synth.S_X)
    X[0, 0, 0, :3] = [0.0, -0.0, 1e-30]
    dY = synth.uniform(X.shape, 2, synth.S_DY)
    td = torch.bfloat16 if dtype == "bf16" else torch.float32
    xt = cuda(X).to(td)
    Xq = host(xt)
    Y = cb.relu_forward(xt)
    np.testing.assert_array_equal(host(Y), oracle.relu_forward(Xq))
    assert not np.signbit(host(Y)).any()
    dX = cb.relu_backward(xt, cuda(dY).to(td))
    np.testing.assert_array_equal(host(dX), oracle.relu_backward(Xq, host(cuda(dY).to(td))))
    y2 = xt.clone()
    cb.relu_forward(y2, inplace=True)
    np.testing.assert_array_equal(host(y2), host(Y))


POOLS = [((2, 3, 11, 11), (3, 3), (2, 2), (0, 0)), ((2, 4, 8, 8), (2, 2), (2, 2), (0, 0)),
         ((1, 2, 7, 6), (3, 3), (2, 2), (1, 1)), ((2, 96, 55, 55), (3, 3), (2, 2), (0, 0))]


@pytest.mark.parametrize("case", POOLS)
def test_maxpool_bit_exact(oracle, case):
    import paper_1408_5093_b200 as cb
    shape, k, s, p = case
    X = synth.uniform(shape, 3, synth.S_X)
    X[0, 0] = np.round(X[0, 0] * 2)  # plenty of ties in one plane (R7)
    Y, M = cb.pool_forward(cuda(X), "max", k, s, p)
    rY, rM = oracle.maxpool_forward(X, k, s, p)
    np.testing.assert_array_equal(host(Y), rY)
    np.testing.assert_array_equal(host(M), rM)
    dY = synth.uniform(rY.shape, 3, synth.S_DY)
    dX = cb.pool_backward(cuda(dY), M, shape, "max", k, s, p)
    np.testing.assert_array_equal(host(dX), oracle.maxpool_backward(dY, rM, shape, k, s, p))


@pytest.mark.parametrize("case", POOLS[:3])
def test_avepool(oracle, case):
    import paper_1408_5093_b200 as cb
    shape, k, s, p = case
    X = synth.uniform(shape, 4, synth.S_X)
    Y, _ = cb.pool_forward(cuda(X), "ave", k, s, p)
    assert_fp32_close(host(Y), oracle.avepool_forward(X, k, s, p), "avepool fwd")
    dY = synth.uniform(tuple(Y.shape), 4, synth.S_DY)
    dX = cb.pool_backward(cuda(dY), None, shape, "ave", k, s, p)
    assert_fp32_close(host(dX), oracle.avepool_backward(dY, shape, k, s, p), "avepool bwd")


@pytest.mark.parametrize("case", [POOLS[0], POOLS[2], POOLS[3]])
@pytest.mark.parametrize("layout", ["nchw_f32", "nhwc_bf16"])
def test_pool_relu_backward_fused(oracle, case, layout):
    """caffe_pool_relu_backward == oracle relu_backward(maxpool_backward(.)) bit for bit, on a
    ReLU output with many exact zeros (whole zero windows included)."""
    import torch
    import paper_1408_5093_b200 as cb
    shape, k, s, p = case
    X = oracle.relu_forward(synth.uniform(shape, 6, synth.S_X) - 0.3)   # ~65% zeros after the ReLU
    if layout == "nhwc_bf16":
        X = oracle.quant_bf16(X)
        xt = cuda(X).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    else:
        xt = cuda(X)
    Y, M = cb.pool_forward(xt, "max", k, s, p)
    rY, rM = oracle.maxpool_forward(X, k, s, p)
    dY = synth.uniform(rY.shape, 6, synth.S_DY)
    if layout == "nhwc_bf16":
        dY = oracle.quant_bf16(dY)
        dyt = cuda(dY).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    else:
        dyt = cuda(dY)
    dX = cb.pool_relu_backward(Y, dyt, M, shape, k, s, p)
    ref = oracle.relu_backward(X, oracle.maxpool_backward(dY, rM, shape, k, s, p))
    if layout == "nhwc_bf16":
        ref = oracle.quant_bf16(ref)
    np.testing.assert_array_equal(host(dX), ref)
    # and it equals the two-kernel sequence through the library
    two = cb.relu_backward(xt, cb.pool_backward(dyt, M, shape, "max", k, s, p))
    np.testing.assert_array_equal(host(dX), host(two))


def test_pool_bf16_maxpool_bit_exact(oracle):
    import torch
    import paper_1408_5093_b200 as cb
    shape, k, s, p = POOLS[0]
    X = oracle.quant_bf16(synth.uniform(shape, 5, synth.S_X))
    Y, M = cb.pool_forward(cuda(X).to(torch.bfloat16), "max", k, s, p)
    rY, rM = oracle.maxpool_forward(X, k, s, p)
    np.testing.assert_array_equal(host(Y), rY)
    np.testing.assert_array_equal(host(M), rM)


@pytest.mark.parametrize("params", [(5, 1e-4, 0.75, 1.0), (3, 0.5, 0.75, 2.0), (5, 2.0, 1.3, 1.0)])
def test_lrn(oracle, params):
    import paper_1408_5093_b200 as cb
    n, a, b, k = params
    X = synth.uniform((2, 9, 5, 6), 6, synth.S_X) * 3
    Y, S = cb.lrn_forward(cuda(X), n, a, b, k, want_scale=True)
    rY, rS = oracle.lrn_forward(X, n, a, b, k, want_scale=True)
    assert_fp32_close(host(Y), rY, "lrn fwd")
    assert_fp32_close(host(S), rS, "lrn scale")
    dY = synth.uniform(X.shape, 6, synth.S_DY)
    ref = oracle.lrn_backward(X, dY, n, a, b, k)
    for sc in (S, None):
        dX = cb.lrn_backward(cuda(X), Y, cuda(dY), n, a, b, k, scale=sc)
        assert_fp32_close(host(dX), ref, "lrn bwd")


IPS = [(4, (3, 2, 5), 7), (64, (50, 4, 4), 500), (64, (500, 1, 1), 10), (256, (256, 6, 6), 300)]


@pytest.mark.parametrize("math", ["fp32", "bf16", "tf32"])
@pytest.mark.parametrize("case", IPS)
def test_inner_product(oracle, case, math):
    import paper_1408_5093_b200 as cb
    N, chw, O = case
    X = synth.uniform((N,) + chw, 7, synth.S_X)
    K = int(np.prod(chw))
    Wt = synth.xavier((O, K), 7)
    b = synth.uniform((O,), 7, synth.S_B)
    dY = synth.uniform((N, O), 7, synth.S_DY)
    q = {"fp32": (lambda v: v), "bf16": oracle.quant_bf16, "tf32": oracle.quant_tf32_rn}[math]
    chk = assert_fp32_close if math == "fp32" else assert_tc_close
    Y = cb.ip_forward(cuda(X), cuda(Wt), cuda(b), math=math)
    chk(host(Y), oracle.ip_forward(q(X), q(Wt), b), "ip fwd")
    Yr = cb.ip_forward(cuda(X), cuda(Wt), cuda(b), math=math, relu=True)
    chk(host(Yr), np.maximum(oracle.ip_forward(q(X), q(Wt), b), 0), "ip fwd relu")
    dX = cb.ip_backward_data(cuda(dY), cuda(Wt), X.shape, math=math)
    rdX, rdW, rdb = oracle.ip_backward(q(X), q(Wt), q(dY))
    chk(host(dX), rdX, "ip dgrad")
    dW, db = cb.ip_backward_weight(cuda(X), cuda(dY), (O, K), math=math)
    chk(host(dW), rdW, "ip wgrad")
    assert_fp32_close(host(db), oracle.ip_backward(X, Wt, dY)[2], "ip bias grad")


def test_softmax_loss(oracle):
    import torch
    import paper_1408_5093_b200 as cb
    s = synth.uniform((256, 1000), 8, synth.S_X) * 5
    lab = synth.labels(256, 1000, 8)
    loss, d = cb.softmax_loss(cuda(s), cuda(lab))
    rl, rd = oracle.softmax_loss(s, lab)
    assert abs(float(loss) - rl) <= 1e-5 * (abs(rl) + 1)
    assert_fp32_close(host(d), rd, "softmax diff")
    loss, _ = cb.softmax_loss(torch.zeros((3, 10), device="cuda"), cuda(np.array([0, 4, 9], np.int32)))
    assert abs(float(loss) - np.log(10)) < 1e-6


def test_sgd(oracle):
    import torch
    import paper_1408_5093_b200 as cb
    w = synth.uniform((1000,), 9, synth.S_W)
    g = synth.uniform((1000,), 9, synth.S_DY)
    v = synth.uniform((1000,), 9, synth.S_AUX) * 0.1
    wt, gt, vt = cuda(w), cuda(g), cuda(v)
    wb = torch.empty(1000, dtype=torch.bfloat16, device="cuda")
    cb.sgd_update(wt, gt, vt, 0.01, 0.9, 5e-4, 0.5, w_bf16=wb)
    rw, rv = oracle.sgd_update(w, g, v, 0.01, 0.9, 5e-4, 0.5)
    assert_fp32_close(host(wt), rw, "sgd w")
    assert_fp32_close(host(vt), rv, "sgd v")
    np.testing.assert_array_equal(host(wb), oracle.quant_bf16(host(wt)))
    w0 = wt.clone()
    cb.sgd_update(wt, gt, torch.zeros_like(vt), 0.0, 0.0, 0.0)  # S:558 zero-LR fixed point
    np.testing.assert_array_equal(host(wt), host(w0))


@pytest.mark.parametrize("case", POOLS)
def test_pool_lrn_relu_nhwc(oracle, case):
    """Channels-last blobs (and mixed in/out layouts) give the same bits as NCHW."""
    import torch
    import paper_1408_5093_b200 as cb
    shape, k, s, p = case
    X = synth.uniform(shape, 11, synth.S_X)
    X[0, 0] = np.round(X[0, 0] * 2)
    cl = torch.channels_last
    xn = cuda(X)
    xh = xn.contiguous(memory_format=cl)
    Yn, Mn = cb.pool_forward(xn, "max", k, s, p)
    Yh, Mh = cb.pool_forward(xh, "max", k, s, p)
    assert cb.layout_of(Yh) == 1 or Yh.shape[2] * Yh.shape[3] == 1
    np.testing.assert_array_equal(host(Yh), host(Yn))
    np.testing.assert_array_equal(host(Mh), host(Mn))
    # NHWC in -> NCHW out
    Yx = torch.empty(tuple(Yn.shape), device="cuda")
    cb.pool_forward(xh, "max", k, s, p, out=Yx, mask=torch.empty(tuple(Yn.shape), dtype=torch.int32, device="cuda"))
    np.testing.assert_array_equal(host(Yx), host(Yn))
    dY = synth.uniform(tuple(Yn.shape), 11, synth.S_DY)
    dXn = cb.pool_backward(cuda(dY), Mn, shape, "max", k, s, p)
    dXh = cb.pool_backward(cuda(dY).contiguous(memory_format=cl), Mh, shape, "max", k, s, p)
    np.testing.assert_array_equal(host(dXh), host(dXn))
    Ya, _ = cb.pool_forward(xh, "ave", k, s, p)
    assert_fp32_close(host(Ya), oracle.avepool_forward(X, k, s, p), "avepool nhwc")
    L = cb.lrn_forward(xh)
    assert_fp32_close(host(L), oracle.lrn_forward(X), "lrn nhwc")
    dXl = cb.lrn_backward(xh, L, cuda(X * 0.5).contiguous(memory_format=cl))
    assert_fp32_close(host(dXl), oracle.lrn_backward(X, X * 0.5), "lrn bwd nhwc")
    R = cb.relu_forward(xh)
    np.testing.assert_array_equal(host(R), oracle.relu_forward(X))


@pytest.mark.parametrize("shape", [(2, 96, 27, 27), (2, 256, 13, 13), (1, 16, 7, 9)])
def test_pool_lrn_nhwc_bf16_vector_paths(oracle, shape):
    """The 8-channel vectorised channels-last BF16 kernels (CaffeNet's layout): max pool values,
    argmax and backward bit-exact; LRN within one BF16 rounding of the fp64 oracle."""
    import torch
    import paper_1408_5093_b200 as cb
    cl = torch.channels_last
    q = oracle.quant_bf16
    X = q(synth.uniform(shape, 14, synth.S_X) * 3)
    X[0, 0] = np.round(X[0, 0])
    xh = cuda(X).to(torch.bfloat16).contiguous(memory_format=cl)
    Y, M = cb.pool_forward(xh, "max", 3, 2)
    rY, rM = oracle.maxpool_forward(X, (3, 3), (2, 2))
    np.testing.assert_array_equal(host(Y), rY)
    np.testing.assert_array_equal(host(M), rM)
    dY = q(synth.uniform(rY.shape, 14, synth.S_DY))
    dX = cb.pool_backward(cuda(dY).to(torch.bfloat16).contiguous(memory_format=cl), M, shape, "max", 3, 2)
    np.testing.assert_array_equal(host(dX), q(oracle.maxpool_backward(dY, rM, shape, (3, 3), (2, 2))))
    for size, a, b, k in ((5, 1e-4, 0.75, 1.0), (3, 0.5, 0.75, 2.0), (9, 2.0, 1.3, 1.0)):
        L, S = cb.lrn_forward(xh, size, a, b, k, want_scale=True)
        rL, rS = oracle.lrn_forward(X, size, a, b, k, want_scale=True)
        assert_bf16_ulp(host(L), rL, f"lrn fwd bf16 nhwc n={size}")
        assert_fp32_close(host(S), rS, "lrn scale")
        G = q(synth.uniform(shape, 15, synth.S_DY))
        dL = cb.lrn_backward(xh, L, cuda(G).to(torch.bfloat16).contiguous(memory_format=cl), size, a, b, k)
        rdL = oracle.lrn_backward(X, G, size, a, b, k)
        assert_tc_close(host(dL), q(rdL.astype(np.float32)), f"lrn bwd bf16 nhwc n={size}")
        # the kernel reads the stored BF16 top in the cross-channel term: admit its rounding where the
        # direct term cancels
        assert_bf16_ulp(host(dL), rdL, f"lrn bwd bf16 nhwc n={size}", atol=float(np.abs(rdL).max()) * 2.0 ** -16)


@pytest.mark.parametrize("shape", [(8, 16, 3, 3, 10), (256, 256, 6, 6, 512)])
def test_ip_nhwc_bottom(oracle, shape):
    """An NHWC bottom is flattened in Caffe's (c,h,w) order.  The pool5->fc6-like case
    (256 x 9216 -> 512) runs the split-K forward and data-gradient with the NHWC scatter, and
    checks beta accumulation into an existing bottom_diff."""
    import torch
    import paper_1408_5093_b200 as cb
    N, C, H, W, O = shape
    K = C * H * W
    X = synth.uniform((N, C, H, W), 12, synth.S_X)
    Wt = synth.xavier((O, K), 12)
    dY = synth.uniform((N, O), 12, synth.S_DY)
    xh = cuda(X).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    Xq = host(xh)
    Y = cb.ip_forward(xh, cuda(Wt), None, math="bf16", out_dtype=torch.float32)
    assert_tc_close(host(Y), oracle.ip_forward(Xq, oracle.quant_bf16(Wt)), "ip fwd nhwc")
    dW, _ = cb.ip_backward_weight(xh, cuda(dY), (O, K), math="bf16")
    rdX, rdW, _ = oracle.ip_backward(Xq, oracle.quant_bf16(Wt), oracle.quant_bf16(dY))
    assert_tc_close(host(dW), rdW, "ip wgrad nhwc")
    dX = torch.zeros((N, C, H, W), device="cuda").contiguous(memory_format=torch.channels_last)
    cb.ip_backward_data(cuda(dY), cuda(Wt), X.shape, math="bf16", out=dX)
    assert_tc_close(host(dX), rdX, "ip dgrad nhwc")
    prev = synth.uniform((N, C, H, W), 13, synth.S_AUX)
    dX2 = cuda(prev).contiguous(memory_format=torch.channels_last)
    cb.ip_backward_data(cuda(dY), cuda(Wt), X.shape, math="bf16", beta=1.0, out=dX2)
    assert_tc_close(host(dX2), rdX + prev, "ip dgrad nhwc beta=1")


@pytest.mark.parametrize("case", POOLS + [((2, 96, 55, 55), (3, 3), (2, 2), (1, 1)), ((1, 16, 9, 11), (2, 3), (1, 2), (1, 1)),
                                  # full 3x3/s2 windows (the specialised kernels), and a clipped last window
                                  ((2, 256, 13, 13), (3, 3), (2, 2), (0, 0)), ((3, 8, 13, 15), (3, 3), (2, 2), (0, 0)),
                                  ((1, 8, 14, 14), (3, 3), (2, 2), (0, 0))])
@pytest.mark.parametrize("layout", ["nchw_f32", "nhwc_bf16"])
def test_maxpool_u8_window_local_mask(oracle, case, layout):
    """A CAFFE_U8 mask holds the same argmax as the int32 mask, as the index local to the unclipped
    window: h*W+w == (py*sh-ph + l//kw)*W + (px*sw-pw + l%kw).  Backward (and the ReLU-fused
    backward) from it equals the oracle bit for bit."""
    import torch
    import paper_1408_5093_b200 as cb
    shape, k, s, p = case
    kh, kw = k
    X = synth.uniform(shape, 16, synth.S_X)
    X[0, 0] = np.round(X[0, 0] * 2)   # ties
    if layout == "nhwc_bf16":
        X = oracle.quant_bf16(X)
        xt = cuda(X).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    else:
        xt = cuda(X)
    Y, M8 = cb.pool_forward(xt, "max", k, s, p, mask_dtype=torch.uint8)
    rY, rM = oracle.maxpool_forward(X, k, s, p)
    np.testing.assert_array_equal(host(Y), rY)
    loc = host(M8).astype(np.int64)
    N, C, OH, OW = rY.shape
    py = np.arange(OH).reshape(1, 1, OH, 1)
    px = np.arange(OW).reshape(1, 1, 1, OW)
    H, W = shape[2], shape[3]
    absidx = (py * s[0] - p[0] + loc // kw) * W + (px * s[1] - p[1] + loc % kw)
    np.testing.assert_array_equal(absidx, rM)
    dY = synth.uniform(rY.shape, 16, synth.S_DY)
    if layout == "nhwc_bf16":
        dY = oracle.quant_bf16(dY)
        dyt = cuda(dY).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    else:
        dyt = cuda(dY)
    dX = cb.pool_backward(dyt, M8, shape, "max", k, s, p)
    ref = oracle.maxpool_backward(dY, rM, shape, k, s, p)
    if layout == "nhwc_bf16":
        ref = oracle.quant_bf16(ref)
    np.testing.assert_array_equal(host(dX), ref)
    dXr = cb.pool_relu_backward(Y, dyt, M8, shape, k, s, p)
    refr = oracle.relu_backward(X, oracle.maxpool_backward(dY, rM, shape, k, s, p))
    if layout == "nhwc_bf16":
        refr = oracle.quant_bf16(refr)
    np.testing.assert_array_equal(host(dXr), refr)


@pytest.mark.parametrize("N,K,O,math,act,nhwc", [
    (256, 4096, 4096, "bf16", "bf16", False),   # fc7 shape: split-K, masked in the reduce
    (256, 4096, 1000, "bf16", "bf16", False),   # fc8 shape
    (8, 96, 40, "bf16", "bf16", False),         # small: direct tensor-core epilogue
    (8, 96, 40, "bf16", "f32", False),          # FP32 output: strided epilogue
    (6, 64, 20, "fp32", "f32", False),          # CUDA-core math: separate ReLU pass
    (4, 32, 24, "bf16", "bf16", True),          # NHWC (C,H,W) bottom: permuted output, separate pass
], ids=["fc7", "fc8", "small", "f32out", "fp32math", "nhwc"])
def test_ip_backward_data_relu(oracle, N, K, O, math, act, nhwc):
    """caffe_ip_backward_data_relu (S:190 + S:208) gives exactly the bits of caffe_ip_backward_data
    followed by the ReLU backward on every reduction / epilogue path, and matches the oracle."""
    import torch
    import paper_1408_5093_b200 as cb
    dt = torch.bfloat16 if act == "bf16" else torch.float32
    shape = (N, K // 8, 2, 4) if nhwc else (N, K)
    top = cuda(synth.uniform(shape, 81, synth.S_X)).to(dt).relu_()
    if nhwc:
        top = top.contiguous(memory_format=torch.channels_last)
    dY = cuda(synth.uniform((N, O), 81, synth.S_DY)).to(dt)
    Wt = cuda(synth.xavier((O, K), 81)).to(torch.bfloat16 if math == "bf16" else torch.float32)
    ref = torch.empty_like(top)
    cb.ip_backward_data(dY, Wt, tuple(top.shape), math=math, out=ref)
    cb.relu_backward(top, ref, inplace=True)
    got = cb.ip_backward_data_relu(dY, Wt, top, math=math)
    np.testing.assert_array_equal(host(got), host(ref))
    qd = oracle.quant_bf16 if math == "bf16" else (lambda a: a)
    rdX, _, _ = oracle.ip_backward(host(top), host(Wt), qd(host(dY)))
    want = oracle.relu_backward(host(top), rdX.reshape(top.shape))
    if act == "bf16":
        rms = float(np.sqrt(np.mean(np.square(want))))
        assert_bf16_ulp(host(got), want, "masked ip dgrad (BF16 out)", atol=rms * 2.0 ** -12)
    elif math == "fp32":
        assert_fp32_close(host(got), want, "masked ip dgrad fp32")
    else:
        assert_tc_close(host(got), want, "masked ip dgrad")
    with pytest.raises(RuntimeError):
        cb.ip_backward_data_relu(dY, Wt, top[:1], math=math)


@pytest.mark.parametrize("N,bshape,O", [
    (256, (256, 4096), 1000),            # fc8: ragged output rows (1000 of 1024)
    (256, (256, 256, 6, 6), 512),        # fc6-like: channels-last (C,H,W) bottom, permuted staging
    (64, (64, 96), 40),                  # small, single-CTA tiles
], ids=["fc8", "fc6like", "small"])
def test_ip_backward_weight_sgd_fused(oracle, N, bshape, O):
    """caffe_ip_backward_weight_sgd (weight gradient consumed by the SGD step in the GEMM epilogue)
    leaves exactly the bits of caffe_ip_backward_weight + caffe_sgd_update in W, the momentum and
    the BF16 copy, writes the same bias gradient, and the update matches the oracle's SGD step."""
    import torch
    import paper_1408_5093_b200 as cb
    x = cuda(synth.uniform(bshape, 91, synth.S_X)).to(torch.bfloat16)
    if len(bshape) == 4:
        x = x.contiguous(memory_format=torch.channels_last)
    K = int(np.prod(bshape[1:]))
    dy = cuda(synth.uniform((N, O), 91, synth.S_DY)).to(torch.bfloat16)
    W0 = cuda(synth.xavier((O, K), 91))
    V0 = cuda(synth.uniform((O, K), 92, synth.S_AUX)) * 0.01
    lr, mom, decay, gs = 0.01, 0.9, 5e-4, 0.5
    # reference: separate gradient + update kernels
    Wr, Vr = W0.clone(), V0.clone()
    Br = torch.empty((O, K), device="cuda", dtype=torch.bfloat16)
    dW, db_r = cb.ip_backward_weight(x, dy, (O, K), beta=0.0)
    cb.sgd_update(Wr, dW, Vr, lr, mom, decay, gs, w_bf16=Br)
    # fused
    Wf, Vf = W0.clone(), V0.clone()
    Bf = torch.empty((O, K), device="cuda", dtype=torch.bfloat16)
    db_f = torch.empty((O,), device="cuda")
    cb.ip_backward_weight_sgd(x, dy, Wf, Vf, Bf, lr, mom, decay, gs, db=db_f)
    np.testing.assert_array_equal(host(Wf), host(Wr))
    np.testing.assert_array_equal(host(Vf), host(Vr))
    np.testing.assert_array_equal(host(Bf), host(Br))
    np.testing.assert_array_equal(host(db_f), host(db_r))
    # and the step itself against the oracle's SGD on the oracle's gradient
    xr = host(x).astype(np.float64).reshape(N, -1)
    g = host(dy).astype(np.float64).T @ xr
    w_o, v_o = oracle.sgd_update(host(W0).astype(np.float64), g, host(V0).astype(np.float64), lr, mom, decay, gs)
    assert_fp32_close(host(Wf), w_o, "fused update: weights")
    assert_fp32_close(host(Vf), v_o, "fused update: momentum")
    assert_tc_close(host(Vf), v_o, "fused update: momentum rel-L2")


@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_blob_to_nchw(dt):
    """caffe_blob_to_nchw: the channels-last blob's elements in NCHW order (BF16 out: bit for bit from
    BF16, RNE from F32); an F32 destination is refused."""
    import torch
    import paper_1408_5093_b200 as cb
    d = torch.bfloat16 if dt == "bf16" else torch.float32
    x = cuda(synth.uniform((5, 256, 6, 6), 111, synth.S_X)).to(d).contiguous(memory_format=torch.channels_last)
    y = cb.to_nchw(x, out=torch.empty(tuple(x.shape), dtype=torch.bfloat16, device="cuda"))
    assert y.is_contiguous()
    np.testing.assert_array_equal(host(y), host(x.to(torch.bfloat16)))
    with pytest.raises(RuntimeError):
        cb.to_nchw(x, out=torch.empty(tuple(x.shape), dtype=torch.float32, device="cuda"))
    with pytest.raises(RuntimeError):
        cb.to_nchw(x, out=torch.empty((5, 256, 6, 5), dtype=d, device="cuda"))


@pytest.mark.parametrize("shape", [(3, 96, 55, 55), (2, 256, 27, 27), (2, 16, 13, 13), (1, 8, 7, 9), (2, 160, 13, 15)],
                         ids=["pool1norm1", "pool2norm2", "c16", "c8odd", "c160"])
@pytest.mark.parametrize("relu", [True, False])
@pytest.mark.parametrize("lrn", [(5, 1e-4, 0.75, 1.0), (3, 0.5, 0.75, 2.0)])
def test_fused_pool_lrn_bit_identical(oracle, shape, relu, lrn):
    """caffe_pool_lrn_forward / caffe_lrn_pool_backward give exactly the bits of
    caffe_pool_forward + caffe_lrn_forward and of caffe_lrn_backward + caffe_pool_(relu_)backward, on
    CaffeNet's pool1/norm1 and pool2/norm2 geometries and small odd ones (ragged strips); and the
    composition matches the oracle (pool bit-exact, LRN within 1 BF16 ulp)."""
    import torch
    import paper_1408_5093_b200 as cb
    cl = torch.channels_last
    size, a, b, k = lrn
    X = oracle.quant_bf16(np.maximum(synth.uniform(shape, 17, synth.S_X) * 4, 0.0) if relu else
                          synth.uniform(shape, 17, synth.S_X) * 4)
    X[0, 0, :4, :4] = 1.0                          # ties
    xt = cuda(X).to(torch.bfloat16).contiguous(memory_format=cl)
    P, M = cb.pool_forward(xt, "max", 3, 2, mask_dtype=torch.uint8)
    Y = cb.lrn_forward(P, size, a, b, k)
    Pf, Mf, Yf = cb.pool_lrn_forward(xt, 3, 2, 0, size, a, b, k)
    np.testing.assert_array_equal(host(Pf), host(P))
    np.testing.assert_array_equal(host(Mf).astype(np.int64), host(M).astype(np.int64))
    np.testing.assert_array_equal(host(Yf), host(Y))
    G = cuda(oracle.quant_bf16(synth.uniform(tuple(P.shape), 18, synth.S_DY))).to(torch.bfloat16) \
        .contiguous(memory_format=cl)
    dP = cb.lrn_backward(P, Y, G, size, a, b, k)
    dX = cb.pool_relu_backward(P, dP, M, shape, 3, 2) if relu else cb.pool_backward(dP, M, shape, "max", 3, 2)
    dXf = cb.lrn_pool_backward(Pf, G, Mf, shape, 3, 2, 0, size, a, b, k, relu=relu)
    np.testing.assert_array_equal(host(dXf), host(dX))
    # against the oracle: pool exact, LRN <= 1 ulp, the pool backward of the GPU's LRN diff exact
    rP, rM = oracle.maxpool_forward(X, (3, 3), (2, 2))
    np.testing.assert_array_equal(host(Pf), rP)
    assert_bf16_ulp(host(Yf), oracle.lrn_forward(rP, size, a, b, k), "fused lrn fwd")
    rdP = oracle.lrn_backward(rP, host(G), size, a, b, k)
    assert_bf16_ulp(host(dP), rdP, "lrn bwd", atol=float(np.abs(rdP).max()) * 2.0 ** -16)
    ref = oracle.maxpool_backward(host(dP), rM, shape, (3, 3), (2, 2))
    if relu:
        ref = oracle.relu_backward(X, ref)
    np.testing.assert_array_equal(host(dXf), oracle.quant_bf16(ref))


def test_fused_pool_lrn_rejects_other_geometry():
    import torch
    import paper_1408_5093_b200 as cb
    x = torch.zeros((1, 16, 12, 12), device="cuda", dtype=torch.bfloat16).contiguous(memory_format=torch.channels_last)
    with pytest.raises(cb.CaffeError, match="E_INVALID"):
        cb.pool_lrn_forward(x, 2, 2, 0)              # 2x2 windows
    with pytest.raises(cb.CaffeError, match="E_DTYPE"):
        cb.pool_lrn_forward(x.float(), 3, 2, 0)


@pytest.mark.parametrize("shape", [(2, 96, 27, 27), (2, 256, 13, 13), (1, 16, 55, 55)])
def test_fp32_nhwc_vector_paths(oracle, shape):
    """FP32 channels-last (the TF32 net's activations): the vector LRN kernels within the FP32 bar of
    the oracle, and the 3x3/s2 max-pool backward (U8 mask, with and without the ReLU gate)
    bit-exact (R8's FP32 gather order)."""
    import torch
    import paper_1408_5093_b200 as cb
    cl = torch.channels_last
    X = synth.uniform(shape, 31, synth.S_X) * 3
    xt = cuda(X).contiguous(memory_format=cl)
    L = cb.lrn_forward(xt)
    assert_fp32_close(host(L), oracle.lrn_forward(X), "lrn fwd f32 nhwc")
    G = synth.uniform(shape, 32, synth.S_DY)
    dL = cb.lrn_backward(xt, L, cuda(G).contiguous(memory_format=cl))
    assert_fp32_close(host(dL), oracle.lrn_backward(X, G), "lrn bwd f32 nhwc")
    Xr = np.maximum(X, 0)
    Xr[0, 0, :3, :3] = 1.0                           # ties
    xr = cuda(Xr).contiguous(memory_format=cl)
    P, M = cb.pool_forward(xr, "max", 3, 2, mask_dtype=torch.uint8)
    rP, rM = oracle.maxpool_forward(Xr, (3, 3), (2, 2))
    np.testing.assert_array_equal(host(P), rP)
    dY = synth.uniform(rP.shape, 33, synth.S_DY)
    dYt = cuda(dY).contiguous(memory_format=cl)
    np.testing.assert_array_equal(host(cb.pool_backward(dYt, M, shape, "max", 3, 2)),
                                  oracle.maxpool_backward(dY, rM, shape, (3, 3), (2, 2)))
    np.testing.assert_array_equal(host(cb.pool_relu_backward(P, dYt, M, shape, 3, 2)),
                                  oracle.relu_backward(Xr, oracle.maxpool_backward(dY, rM, shape, (3, 3), (2, 2))))


@pytest.mark.parametrize("shape", [(5, 256, 6, 6), (3, 64, 4, 6)], ids=["pool5", "C64HW24"])
def test_ip_nhwc_rows_staging_bit_identical(oracle, shape):
    """The (c,h,w) row staging of a channels-last BF16 inner-product input (CAFFE_TUNE_ROWS_CB: one
    block per 64-channel block and image, or one per image) gives the same bits for the forward and
    the weight gradient, and the forward meets the oracle bar (flatten order S:130)."""
    import torch
    import paper_1408_5093_b200 as cb
    from paper_1408_5093_b200 import _abi
    N, C, H, W = shape
    K, O = C * H * W, 96
    x = synth.uniform(shape, 3, synth.S_X)
    w = synth.xavier((O, K), 3)
    dy = synth.uniform((N, O), 3, synth.S_DY)
    xd = cuda(x).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    wd = cuda(w).to(torch.bfloat16)
    outs = []
    try:
        for v in (1, 0):
            _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_ROWS_CB, v)
            y = cb.ip_forward(xd, wd, None, "bf16", out_dtype=torch.float32)
            dw, _ = cb.ip_backward_weight(xd, cuda(dy).to(torch.bfloat16), (O, K), "bf16")
            outs.append((host(y), host(dw)))
    finally:
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_ROWS_CB, 1)
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])
    q = oracle.quant_bf16
    assert_tc_close(outs[0][0], oracle.ip_forward(q(x.reshape(N, -1)), q(w)), "ip fwd nhwc rows")


@pytest.mark.parametrize("N,O", [(256, 4096), (37, 1000), (3, 20)], ids=["fc6", "fc8odd", "tiny"])
def test_ip_bias_grad_one_pass(oracle, N, O):
    """Inner-product bias gradient db = beta*db + sum_n dY in one pass (CAFFE_TUNE_BIAS_ROWS=1)
    and as split partials + final (=0): each meets the FP32 bar against the oracle, both with beta=1
    accumulation, and each is deterministic run to run."""
    import torch
    import paper_1408_5093_b200 as cb
    from paper_1408_5093_b200 import _abi
    K = 64
    x = synth.uniform((N, K), 4, synth.S_X)
    dy = synth.uniform((N, O), 4, synth.S_DY)
    prev = synth.uniform((O,), 4, synth.S_AUX)
    ref = dy.astype(np.float64).sum(0) + prev
    try:
        for v in (1, 0):
            _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_BIAS_ROWS, v)
            got = []
            for _ in range(2):
                db = cuda(prev.copy())
                cb.ip_backward_weight(cuda(x), cuda(dy), (O, K), "bf16", beta=1.0, dw=torch.zeros(O, K, device="cuda"),
                                      db=db)
                got.append(host(db))
            np.testing.assert_array_equal(got[0], got[1])
            assert_fp32_close(got[0], ref, f"ip db bias_rows={v}")
    finally:
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_BIAS_ROWS, 0)


@pytest.mark.parametrize("shape", [(2, 96, 27, 27), (2, 256, 13, 13), (3, 16, 5, 7), (1, 160, 6, 6)])
@pytest.mark.parametrize("size", [5, 3, 9])
def test_lrn_backward_c16_bit_identical(oracle, shape, size):
    """The 16-channel-lane BF16 LRN backward (CAFFE_TUNE_LRN_BWD_C16, neighbours by shuffle) writes
    exactly the bits of the 8-channel kernel, and meets the BF16 bar against the oracle."""
    import torch
    import paper_1408_5093_b200 as cb
    from paper_1408_5093_b200 import _abi
    cl = torch.channels_last
    x = oracle.quant_bf16(synth.uniform(shape, 23, synth.S_X) * 3)
    g = oracle.quant_bf16(synth.uniform(shape, 23, synth.S_DY))
    xd = cuda(x).to(torch.bfloat16).contiguous(memory_format=cl)
    gd = cuda(g).to(torch.bfloat16).contiguous(memory_format=cl)
    y = cb.lrn_forward(xd, local_size=size)
    outs = []
    try:
        for v in (1, 0):
            _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_LRN_BWD_C16, v)
            outs.append(host(cb.lrn_backward(xd, y, gd, local_size=size).float()))
    finally:
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_LRN_BWD_C16, 1)
    np.testing.assert_array_equal(outs[0], outs[1])
    ref = oracle.lrn_backward(x.astype(np.float64), g.astype(np.float64), size=size, alpha=1e-4, beta=0.75, k=1.0)
    assert_bf16_ulp(outs[0], ref, f"lrn bwd c16 size={size}", atol=float(np.abs(ref).max()) * 2.0 ** -16)
