"""GPU parity of the convolution ABI calls against the CPU oracle (-m gpu).

FP32 math: per-element |err| <= 1e-5(|ref|+1).  BF16/TF32 math: relative L2 <= 1e-3 against the
oracle fed the same RNE-quantized operands (reading R12); results are FP32.
"""
import numpy as np
import pytest

import synth
from _helpers import assert_bf16_ulp, assert_fp32_close, assert_tc_close, cuda, host

pytestmark = pytest.mark.gpu

# N, C, H, W, O, k, s, p, g  -- spans several M tiles, ragged tails, groups, stride (s2d path)
CASES = [
    (2, 3, 9, 9, 8, (3, 3), (1, 1), (1, 1), 1),
    (3, 8, 13, 13, 12, (3, 3), (1, 1), (1, 1), 2),        # conv4/5-like, 2 groups, ragged M
    (2, 6, 27, 27, 32, (5, 5), (1, 1), (2, 2), 2),        # conv2-like, Cg=3 (K padding)
    (2, 3, 35, 35, 16, (11, 11), (4, 4), (0, 0), 1),      # conv1-like, stride 4 (s2d path)
    (2, 1, 28, 28, 20, (5, 5), (1, 1), (0, 0), 1),        # LeNet conv1
    (2, 20, 12, 12, 50, (5, 5), (1, 1), (0, 0), 1),       # LeNet conv2
    (1, 4, 10, 9, 6, (3, 2), (2, 1), (1, 0), 2),          # asymmetric stride/kernel/pad
    (2, 128, 13, 13, 96, (3, 3), (1, 1), (1, 1), 1),      # several channel blocks (Cg=128)
    (1, 72, 8, 8, 300, (1, 1), (1, 1), (0, 0), 1),        # 1x1, 2 N tiles
]
IDS = [f"N{c[0]}C{c[1]}H{c[2]}O{c[4]}k{c[5][0]}s{c[6][0]}p{c[7][0]}g{c[8]}" for c in CASES]


def _inputs(case, seed=0):
    N, C, H, W, O, k, s, p, g = case
    X = synth.uniform((N, C, H, W), seed, synth.S_X)
    Wt = synth.xavier((O, C // g) + k, seed)
    b = synth.uniform((O,), seed, synth.S_B)
    OH = (H + 2 * p[0] - k[0]) // s[0] + 1
    OW = (W + 2 * p[1] - k[1]) // s[1] + 1
    dY = synth.uniform((N, O, OH, OW), seed, synth.S_DY)
    return X, Wt, b, dY


def _atol(ref):
    """Absolute slack of a per-element BF16-ulp check where the exact result cancels to ~0: 2^-12 of
    the RMS output (the FP32 accumulation error of the long dot products, not a BF16 spacing)."""
    return float(np.sqrt(np.mean(np.square(ref)))) * 2.0 ** -12


def _quant(oracle, math, a):
    return {"fp32": lambda v: v, "bf16": oracle.quant_bf16, "tf32": oracle.quant_tf32_rn}[math](a)


@pytest.mark.parametrize("math", ["fp32", "bf16", "tf32"])
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_conv_forward(oracle, case, math):
    import paper_1408_5093_b200 as cb
    N, C, H, W, O, k, s, p, g = case
    X, Wt, b, _ = _inputs(case)
    for relu in (False, True):
        Y = cb.conv_forward(cuda(X), cuda(Wt), cuda(b), stride=s, pad=p, group=g, math=math, relu=relu)
        ref = oracle.conv_forward(_quant(oracle, math, X), _quant(oracle, math, Wt), b, stride=s, pad=p, group=g,
                                  relu=relu)
        if math == "fp32":
            assert_fp32_close(host(Y), ref, f"conv fwd relu={relu}")
        else:
            assert_tc_close(host(Y), ref, f"conv fwd {math} relu={relu}")


@pytest.mark.parametrize("math", ["fp32", "bf16", "tf32"])
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_conv_backward_data(oracle, case, math):
    import paper_1408_5093_b200 as cb
    N, C, H, W, O, k, s, p, g = case
    X, Wt, _, dY = _inputs(case, 1)
    dX = cb.conv_backward_data(cuda(dY), cuda(Wt), X.shape, stride=s, pad=p, group=g, math=math)
    ref = oracle.conv_backward_data(_quant(oracle, math, dY), _quant(oracle, math, Wt), X.shape, stride=s, pad=p,
                                    group=g)
    if math == "fp32":
        assert_fp32_close(host(dX), ref, "conv dgrad")
    else:
        assert_tc_close(host(dX), ref, f"conv dgrad {math}")
    # beta = 1 accumulates (S:292 2x rule up to rounding)
    dX0 = synth.uniform(X.shape, 1, synth.S_AUX)
    dX2 = cb.conv_backward_data(cuda(dY), cuda(Wt), X.shape, stride=s, pad=p, group=g, math=math, beta=1.0,
                                out=cuda(dX0))
    if math == "fp32":
        assert_fp32_close(host(dX2), ref + dX0, "conv dgrad beta=1")
    else:
        assert_tc_close(host(dX2), ref + dX0, "conv dgrad beta=1")


@pytest.mark.parametrize("math", ["fp32", "bf16", "tf32"])
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_conv_backward_weight(oracle, case, math):
    import paper_1408_5093_b200 as cb
    N, C, H, W, O, k, s, p, g = case
    X, Wt, _, dY = _inputs(case, 2)
    dW, db = cb.conv_backward_weight(cuda(X), cuda(dY), Wt.shape, stride=s, pad=p, group=g, math=math)
    rW, rb = oracle.conv_backward_weight(_quant(oracle, math, X), _quant(oracle, math, dY), Wt.shape, stride=s, pad=p,
                                         group=g)
    _, rb_exact = oracle.conv_backward_weight(X, dY, Wt.shape, stride=s, pad=p, group=g)
    assert_fp32_close(host(db), rb_exact, "bias grad (fp32 sum of dY)")
    if math == "fp32":
        assert_fp32_close(host(dW), rW, "conv wgrad")
    else:
        assert_tc_close(host(dW), rW, f"conv wgrad {math}")
    # accumulate: beta=1 on top of the previous result gives 2x
    dW2, db2 = cb.conv_backward_weight(cuda(X), cuda(dY), Wt.shape, stride=s, pad=p, group=g, math=math, beta=1.0,
                                       dw=dW.clone(), db=db.clone())
    np.testing.assert_array_equal(host(dW2), 2 * host(dW))
    np.testing.assert_array_equal(host(db2), 2 * host(db))


@pytest.mark.parametrize("math", ["bf16", "fp32"])
def test_conv_deterministic(math):
    """bitwise reproducible run to run."""
    import paper_1408_5093_b200 as cb
    case = CASES[2]
    N, C, H, W, O, k, s, p, g = case
    X, Wt, b, dY = _inputs(case, 3)
    outs = []
    for _ in range(2):
        Y = cb.conv_forward(cuda(X), cuda(Wt), cuda(b), stride=s, pad=p, group=g, math=math)
        dX = cb.conv_backward_data(cuda(dY), cuda(Wt), X.shape, stride=s, pad=p, group=g, math=math)
        dW, db = cb.conv_backward_weight(cuda(X), cuda(dY), Wt.shape, stride=s, pad=p, group=g, math=math)
        outs.append([host(t) for t in (Y, dX, dW, db)])
    for a, b_ in zip(*outs):
        np.testing.assert_array_equal(a, b_)


def test_conv_bf16_storage_output_is_rne_of_fp32(oracle):
    """BF16-output epilogue: bf16 result == RNE(fp32 result), bit-exact."""
    import torch
    import paper_1408_5093_b200 as cb
    case = CASES[1]
    N, C, H, W, O, k, s, p, g = case
    X, Wt, b, _ = _inputs(case, 4)
    Y32 = cb.conv_forward(cuda(X), cuda(Wt), cuda(b), stride=s, pad=p, group=g, math="bf16")
    Y16 = cb.conv_forward(cuda(X), cuda(Wt), cuda(b), stride=s, pad=p, group=g, math="bf16", out_dtype=torch.bfloat16)
    np.testing.assert_array_equal(host(Y16), oracle.quant_bf16(host(Y32)))


def test_conv_empty_batch_is_noop():
    import torch
    import paper_1408_5093_b200 as cb
    X = torch.zeros((0, 3, 8, 8), device="cuda")
    Wt = torch.zeros((4, 3, 3, 3), device="cuda")
    Y = cb.conv_forward(X, Wt, None, pad=1, math="bf16")
    assert Y.shape == (0, 4, 8, 8)


# ---------------------------------------------------------------- channels-last (NHWC) BF16 blobs:
# the tensor-core path reads/writes them directly (no transpose), the FP32 path via strides.
NHWC_CASES = [CASES[1], CASES[2], CASES[3], CASES[7], (2, 16, 9, 9, 24, (3, 3), (1, 1), (1, 1), 2),
              (1, 4, 10, 9, 6, (3, 2), (2, 1), (1, 0), 1),    # padded s2d from a channels-last image
              CASES[6]]                                        # the same, grouped


@pytest.mark.parametrize("math", ["bf16", "fp32"])
@pytest.mark.parametrize("case", NHWC_CASES, ids=[f"N{c[0]}C{c[1]}H{c[2]}O{c[4]}k{c[5][0]}g{c[8]}" for c in NHWC_CASES])
def test_conv_nhwc_bf16_storage(oracle, case, math):
    import torch
    import paper_1408_5093_b200 as cb
    N, C, H, W, O, k, s, p, g = case
    X, Wt, b, dY = _inputs(case, 5)
    cl = torch.channels_last
    Xd = cuda(X).to(torch.bfloat16).contiguous(memory_format=cl)
    dYd = cuda(dY).to(torch.bfloat16).contiguous(memory_format=cl)
    Xq, dYq = host(Xd), host(dYd)
    Wq = oracle.quant_bf16(Wt) if math == "bf16" else Wt
    chk = assert_tc_close if math == "bf16" else (lambda a, r, w: assert_fp32_close(a, r, w))
    Y = cb.conv_forward(Xd, cuda(Wt), cuda(b), stride=s, pad=p, group=g, math=math, relu=True, out_dtype=torch.float32)
    assert cb.layout_of(Y) == 1 or min(Y.shape[1], Y.shape[2] * Y.shape[3]) == 1
    chk(host(Y), oracle.conv_forward(Xq, Wq, b, stride=s, pad=p, group=g, relu=True), "fwd nhwc")
    dX = cb.conv_backward_data(dYd, cuda(Wt), X.shape, stride=s, pad=p, group=g, math=math, out_dtype=torch.float32)
    chk(host(dX), oracle.conv_backward_data(dYq, Wq, X.shape, stride=s, pad=p, group=g), "dgrad nhwc")
    dW, db = cb.conv_backward_weight(Xd, dYd, Wt.shape, stride=s, pad=p, group=g, math=math)
    rW, rb = oracle.conv_backward_weight(Xq, dYq, Wt.shape, stride=s, pad=p, group=g)
    chk(host(dW), rW, "wgrad nhwc")
    assert_fp32_close(host(db), rb, "bias grad nhwc")
    # bf16 NHWC output epilogue == RNE of the fp32 result (vectorised row stores)
    Y16 = cb.conv_forward(Xd, cuda(Wt), cuda(b), stride=s, pad=p, group=g, math=math, relu=True)
    np.testing.assert_array_equal(host(Y16), oracle.quant_bf16(host(Y)))


@pytest.mark.parametrize("cta", [1, 2])
@pytest.mark.parametrize("case", CASES + [(4, 64, 27, 27, 192, (3, 3), (1, 1), (1, 1), 1)],
                         ids=IDS + ["N4C64H27O192"])
def test_conv_cta_pair_modes(oracle, case, cta):
    """The single-CTA (M=128) and CTA-pair (tcgen05 cta_group::2, M=256) tensor-core tiles give the
    same parity for forward and data gradient, for every geometry (forced via caffe_set_tuning)."""
    import torch
    import paper_1408_5093_b200 as cb
    from paper_1408_5093_b200 import _abi
    N, C, H, W, O, k, s, p, g = case
    X, Wt, b, dY = _inputs(case, 6)
    q = oracle.quant_bf16
    cl = torch.channels_last
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_CTA_PAIR, cta)
    try:
        Xd = cuda(X).to(torch.bfloat16).contiguous(memory_format=cl)
        Y = cb.conv_forward(Xd, cuda(Wt), cuda(b), stride=s, pad=p, group=g, relu=True, out_dtype=torch.float32)
        assert_tc_close(host(Y), oracle.conv_forward(host(Xd), q(Wt), b, stride=s, pad=p, group=g, relu=True),
                        f"fwd cta={cta}")
        dX = cb.conv_backward_data(cuda(dY), cuda(Wt), X.shape, stride=s, pad=p, group=g)
        assert_tc_close(host(dX), oracle.conv_backward_data(q(dY), q(Wt), X.shape, stride=s, pad=p, group=g),
                        f"dgrad cta={cta}")
    finally:
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_CTA_PAIR, 0)


@pytest.mark.parametrize("macc", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("case", [CASES[2], CASES[3], CASES[7], (2, 64, 13, 13, 192, (3, 3), (1, 1), (1, 1), 2)],
                         ids=[IDS[2], IDS[3], IDS[7], "N2C64H13O192g2"])
def test_conv_wgrad_multi_accumulator(oracle, case, macc):
    """Weight gradient with 1..4 M tiles per work unit (top_diff staged once per unit; forced via
    CAFFE_TUNE_WGRAD_MACC, 0 = automatic): same parity for every count, ragged last unit included."""
    import torch
    import paper_1408_5093_b200 as cb
    from paper_1408_5093_b200 import _abi
    N, C, H, W, O, k, s, p, g = case
    X, Wt, b, dY = _inputs(case, 9)
    q = oracle.quant_bf16
    cl = torch.channels_last
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_WGRAD_MACC, macc)
    try:
        Xd = cuda(X).to(torch.bfloat16).contiguous(memory_format=cl)
        dYd = cuda(dY).to(torch.bfloat16).contiguous(memory_format=cl)
        dW, db = cb.conv_backward_weight(Xd, dYd, Wt.shape, stride=s, pad=p, group=g, math="bf16")
        rW, rb = oracle.conv_backward_weight(host(Xd), host(dYd), Wt.shape, stride=s, pad=p, group=g)
        assert_tc_close(host(dW), rW, f"wgrad macc={macc}")
        assert_fp32_close(host(db), rb, f"bias grad macc={macc}")
    finally:
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_WGRAD_MACC, 0)


@pytest.mark.parametrize("dy_layout", ["nchw_f32", "nhwc_f32", "nhwc_bf16"])
def test_caffenet_conv1_full_image_wgrad(oracle, dy_layout):
    """conv1 at its real geometry (227x227, 11x11/s4, space-to-depth path), 2 images, every dY layout."""
    import torch
    import paper_1408_5093_b200 as cb
    X = synth.int_pixels((2, 3, 227, 227), 13)
    Wt = synth.gaussian((96, 3, 11, 11), 0.01, 13)
    dY = synth.uniform((2, 96, 55, 55), 13, synth.S_DY)
    dYd = cuda(dY)
    if dy_layout != "nchw_f32":
        dYd = dYd.contiguous(memory_format=torch.channels_last)
    if dy_layout == "nhwc_bf16":
        dYd = dYd.to(torch.bfloat16)
    dW, db = cb.conv_backward_weight(cuda(X), dYd, Wt.shape, stride=4, pad=0, group=1, math="bf16")
    rW, _ = oracle.conv_backward_weight(X, oracle.quant_bf16(dY), Wt.shape, stride=(4, 4))
    assert_tc_close(host(dW), rW, f"conv1 wgrad {dy_layout}")
    Y = cb.conv_forward(cuda(X), cuda(Wt), None, stride=4, math="bf16")
    rY = oracle.conv_forward(X, oracle.quant_bf16(Wt), None, stride=(4, 4))
    assert_tc_close(host(Y), rY, "conv1 fwd")
    # channels-last bf16 image batch (the training net's input blob): the direct s2d pack
    Xh = cuda(X).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)   # integer pixels: exact
    Yh = cb.conv_forward(Xh, cuda(Wt), None, stride=4, math="bf16")
    np.testing.assert_array_equal(host(Yh), host(cb.conv_forward(cuda(X), cuda(Wt), None, stride=4, math="bf16")
                                                  .to(torch.bfloat16).contiguous(memory_format=torch.channels_last)))


HALO_CASES = CASES + [(2, 96, 27, 27, 64, (5, 5), (1, 1), (2, 2), 2),     # conv2 geometry (Cg=48, K padding)
                      (1, 3, 227, 227, 32, (11, 11), (4, 4), (0, 0), 1),  # conv1 geometry (s2d, 55x55 out)
                      (2, 64, 20, 37, 48, (3, 3), (1, 1), (1, 1), 1),     # ragged last tile rows
                      (2, 256, 13, 13, 192, (3, 3), (1, 1), (1, 1), 2),   # conv4-like: 2 channel blocks, BN 96
                      (2, 384, 13, 13, 128, (3, 3), (1, 1), (1, 1), 2)]   # conv5-like: 3 channel blocks, BN 64
HALO_IDS = IDS + ["conv2geom", "conv1geom", "H20W37", "conv4like", "conv5like"]


@pytest.mark.parametrize("cta", [1, 2])
@pytest.mark.parametrize("halo", [1, 2])
@pytest.mark.parametrize("case", HALO_CASES, ids=HALO_IDS)
def test_conv_halo_tiles(oracle, case, halo, cta):
    """Stride-1 forward / data gradient with halo tiles (one staged input window per channel block,
    row-shifted descriptors per tap; CAFFE_TUNE_HALO=2 forces them wherever the geometry allows,
    1 = per-tap im2col tiles) give the same parity, single-CTA and CTA-pair, NHWC bf16 operands."""
    import torch
    import paper_1408_5093_b200 as cb
    from paper_1408_5093_b200 import _abi
    N, C, H, W, O, k, s, p, g = case
    X, Wt, b, dY = _inputs(case, 11)
    if C == 3 and H == 227:
        X = synth.int_pixels((N, C, H, W), 11)
    q = oracle.quant_bf16
    cl = torch.channels_last
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO, halo)
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_CTA_PAIR, cta)
    try:
        Xd = cuda(X).to(torch.bfloat16).contiguous(memory_format=cl)
        Y = cb.conv_forward(Xd, cuda(Wt), cuda(b), stride=s, pad=p, group=g, relu=True, out_dtype=torch.float32)
        assert_tc_close(host(Y), oracle.conv_forward(host(Xd), q(Wt), b, stride=s, pad=p, group=g, relu=True),
                        f"fwd halo={halo} cta={cta}")
        dYd = cuda(dY).to(torch.bfloat16).contiguous(memory_format=cl)
        if cta == 1:   # weight gradient (single-CTA kernel): halo along the pixel reduction
            dW, db = cb.conv_backward_weight(Xd, dYd, Wt.shape, stride=s, pad=p, group=g, math="bf16")
            rW, rb = oracle.conv_backward_weight(host(Xd), host(dYd), Wt.shape, stride=s, pad=p, group=g)
            assert_tc_close(host(dW), rW, f"wgrad halo={halo}")
            assert_fp32_close(host(db), rb, f"bias grad halo={halo}")
            dW2, _ = cb.conv_backward_weight(Xd, dYd, Wt.shape, stride=s, pad=p, group=g, math="bf16", beta=1.0,
                                             dw=dW.clone(), db=db.clone())
            np.testing.assert_array_equal(host(dW2), 2 * host(dW))
        if C == 3 and H == 227:
            return   # the first layer has no data gradient in the net (and its s2d dgrad is not halo-tiled)
        dX = torch.empty((N, C, H, W), device="cuda").contiguous(memory_format=cl)
        cb.conv_backward_data(dYd, cuda(Wt), X.shape, stride=s, pad=p, group=g, out=dX)
        assert_tc_close(host(dX), oracle.conv_backward_data(host(dYd), q(Wt), X.shape, stride=s, pad=p, group=g),
                        f"dgrad halo={halo} cta={cta}")
        # beta accumulation through the halo epilogue
        prev = synth.uniform(X.shape, 12, synth.S_AUX)
        dX2 = cuda(prev).contiguous(memory_format=cl)
        cb.conv_backward_data(dYd, cuda(Wt), X.shape, stride=s, pad=p, group=g, beta=1.0, out=dX2)
        assert_tc_close(host(dX2), oracle.conv_backward_data(host(dYd), q(Wt), X.shape, stride=s, pad=p, group=g) + prev,
                        f"dgrad beta=1 halo={halo} cta={cta}")
    finally:
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO, 0)
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_CTA_PAIR, 0)


@pytest.mark.parametrize("case", [CASES[7], (2, 64, 13, 13, 256, (3, 3), (1, 1), (1, 1), 2),
                                  (2, 128, 13, 13, 384, (3, 3), (1, 1), (1, 1), 1),
                                  (2, 96, 27, 27, 64, (5, 5), (1, 1), (2, 2), 2), CASES[3]],
                         ids=["C128O96", "C64O256g2", "C128O384", "conv2geom", "conv1like"])
def test_tma_store_epilogue_bit_identical(oracle, case):
    """The TMA-store and row-staged epilogues (CAFFE_TUNE_TMA_STORE, on by default /
    CAFFE_TUNE_ROWS_EPILOGUE, off by default) write exactly what the per-thread direct-store epilogue writes: conv forward
    (bias+ReLU, NHWC bf16 and fp32 out; im2col and halo tiles), data gradient, inner product
    forward / data / weight gradient; and match the oracle."""
    import torch
    import paper_1408_5093_b200 as cb
    from paper_1408_5093_b200 import _abi
    N, C, H, W, O, k, s, p, g = case
    X, Wt, b, dY = _inputs(case, 21)
    cl = torch.channels_last
    Xd = cuda(X).to(torch.bfloat16).contiguous(memory_format=cl)
    dYd = cuda(dY).to(torch.bfloat16).contiguous(memory_format=cl)
    K = C * H * W
    Wip = cuda(synth.xavier((512, K), 21)).to(torch.bfloat16)
    dYip = cuda(synth.uniform((N, 512), 21, synth.S_DY)).to(torch.bfloat16)
    outs = {}
    try:
        for mode in (0, 1, 2):
            _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_TMA_STORE, 1 if mode == 1 else 0)
            _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_ROWS_EPILOGUE, 0 if mode == 0 else 1)
            r = {}
            r["y16"] = cb.conv_forward(Xd, cuda(Wt), cuda(b), stride=s, pad=p, group=g, relu=True)
            r["y32"] = cb.conv_forward(Xd, cuda(Wt), cuda(b), stride=s, pad=p, group=g, relu=True,
                                       out_dtype=torch.float32)
            dX = torch.empty((N, C, H, W), device="cuda", dtype=torch.bfloat16).contiguous(memory_format=cl)
            cb.conv_backward_data(dYd, cuda(Wt), X.shape, stride=s, pad=p, group=g, out=dX)
            r["dx"] = dX
            rows = Xd.permute(0, 2, 3, 1).reshape(N, -1).contiguous()   # any (N, K) bf16 rows
            r["ip"] = cb.ip_forward(rows, Wip, None)
            r["ipd"] = cb.ip_backward_data(dYip, Wip, (N, K, 1, 1))
            r["ipw"], _ = cb.ip_backward_weight(rows, dYip, (512, K))
            outs[mode] = {kk: host(v) for kk, v in r.items()}
    finally:
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_TMA_STORE, 1)
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_ROWS_EPILOGUE, 0)
    for kk in outs[0]:
        np.testing.assert_array_equal(outs[0][kk], outs[1][kk], err_msg=kk)
        np.testing.assert_array_equal(outs[0][kk], outs[2][kk], err_msg=kk)
    q = oracle.quant_bf16
    assert_tc_close(outs[1]["y32"], oracle.conv_forward(host(Xd), q(Wt), b, stride=s, pad=p, group=g, relu=True),
                    "fwd tma store")
    rdx = oracle.conv_backward_data(host(dYd), q(Wt), X.shape, stride=s, pad=p, group=g)
    assert_bf16_ulp(outs[1]["dx"], rdx, "dgrad tma store (BF16 out)", atol=_atol(rdx))


@pytest.mark.parametrize("case", [CASES[3], CASES[6], CASES[1]], ids=[IDS[3], IDS[6], IDS[1]])
def test_conv_prepacked_bottom(oracle, case):
    """caffe_conv_pack_bottom + CAFFE_BOTTOM_PREPACKED on a dedicated workspace give the same bits
    as packing inside each call (forward and weight gradient), for packed (s2d, NCHW) and direct
    operands."""
    import torch
    import paper_1408_5093_b200 as cb
    N, C, H, W, O, k, s, p, g = case
    X, Wt, b, dY = _inputs(case, 31)
    for xt in (cuda(X), cuda(X).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)):
        w = cuda(Wt).to(torch.bfloat16)
        ws = cb.conv_bottom_workspace(X.shape, Wt.shape, s, p, g, "bf16")
        cb.conv_pack_bottom(xt, w, s, p, g, "bf16", ws=ws)
        y1 = cb.conv_forward(xt, w, cuda(b), s, p, g, relu=True, ws=ws, prepacked=True, out_dtype=torch.float32)
        y0 = cb.conv_forward(xt, w, cuda(b), s, p, g, relu=True, out_dtype=torch.float32)
        np.testing.assert_array_equal(host(y1), host(y0))
        dyt = cuda(dY) if xt.dtype == torch.float32 else cuda(dY).to(torch.bfloat16).contiguous(
            memory_format=torch.channels_last)
        dw1, db1 = cb.conv_backward_weight(xt, dyt, Wt.shape, s, p, g, ws=ws, prepacked=True)
        dw0, db0 = cb.conv_backward_weight(xt, dyt, Wt.shape, s, p, g)
        np.testing.assert_array_equal(host(dw1), host(dw0))
        np.testing.assert_array_equal(host(db1), host(db0))


@pytest.mark.parametrize("case", [(2, 3, 67, 67, 96, (11, 11), (4, 4), (0, 0), 1),      # conv1 geometry: 48 cols/group
                                  (2, 96, 27, 27, 256, (5, 5), (1, 1), (2, 2), 2),      # conv2: fwd 64, dgrad 24
                                  (3, 64, 20, 20, 96, (3, 3), (1, 1), (1, 1), 1)],      # fwd 48, dgrad 64 (K=96 -> 2 blocks)
                         ids=["conv1geom", "conv2geom", "C64O96"])
def test_halo_fast_epilogue_bit_identical(oracle, case):
    """The specialised BF16 channels-last halo epilogue (CAFFE_TUNE_HALO_FAST_EPI, default on), with
    direct 16-byte stores or shared-memory staging + 4-D TMA tensor stores (CAFFE_TUNE_HALO_TMA_STORE,
    default off; swizzled 32/128-byte and unswizzled 48-byte box rows), writes exactly the bits of
    the generic per-chunk epilogue (bias + ReLU forward, data gradient), CTA
    pairs with two accumulators per unit, and matches the oracle."""
    import torch
    import paper_1408_5093_b200 as cb
    from paper_1408_5093_b200 import _abi
    N, C, H, W, O, k, s, p, g = case
    X, Wt, b, dY = _inputs(case, 41)
    if C == 3:
        X = synth.int_pixels((N, C, H, W), 41)
    cl = torch.channels_last
    Xd = cuda(X).to(torch.bfloat16).contiguous(memory_format=cl)
    dYd = cuda(dY).to(torch.bfloat16).contiguous(memory_format=cl)
    outs = {}
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO, 2)
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_CTA_PAIR, 2)
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_JN, 0)   # the per-tap kernel's epilogues
    try:
        # generic; specialised with per-row stores; with TMA stores; with warp-transposed coalesced
        # stores; three epilogue groups (the 96-column first layer) coalesced / per-row; four, coalesced
        for fast in (0, 1, 2, 3, 4, 5, 6):
            _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_FAST_EPI, 1 if fast else 0)
            _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_TMA_STORE, 1 if fast == 2 else 0)
            _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_COALESCE, 1 if fast in (3, 4, 6) else 0)
            _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_EPI_GROUPS, {4: 3, 5: 3, 6: 4}.get(fast, 2))
            y = cb.conv_forward(Xd, cuda(Wt), cuda(b), stride=s, pad=p, group=g, relu=True)
            y0 = cb.conv_forward(Xd, cuda(Wt), None, stride=s, pad=p, group=g, relu=False)
            r = {"y": host(y), "y_nobias": host(y0)}
            if s[0] == 1:
                dX = torch.empty((N, C, H, W), device="cuda", dtype=torch.bfloat16).contiguous(memory_format=cl)
                cb.conv_backward_data(dYd, cuda(Wt), X.shape, stride=s, pad=p, group=g, out=dX)
                r["dx"] = host(dX)
            outs[fast] = r
        # same tiles, FP32 output (generic epilogue): the BF16 outputs must be its RNE rounding (R12)
        y32 = cb.conv_forward(Xd, cuda(Wt), cuda(b), stride=s, pad=p, group=g, relu=True, out_dtype=torch.float32)
        dX32 = torch.empty((N, C, H, W), device="cuda").contiguous(memory_format=cl)
        if s[0] == 1:
            cb.conv_backward_data(dYd, cuda(Wt), X.shape, stride=s, pad=p, group=g, out=dX32)
    finally:
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_FAST_EPI, 1)
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_TMA_STORE, 0)
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_COALESCE, 1)
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_EPI_GROUPS, 0)
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO, 0)
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_CTA_PAIR, 0)
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_JN, 1)
    for kk in outs[0]:
        for f in range(1, 7):
            np.testing.assert_array_equal(outs[0][kk], outs[f][kk], err_msg=f"{kk} mode {f}")
    # the BF16 outputs are the RNE rounding of the FP32-output pass (R12), which meets the oracle bar
    q = oracle.quant_bf16
    np.testing.assert_array_equal(outs[1]["y"], host(y32.to(torch.bfloat16)))
    assert_tc_close(host(y32), oracle.conv_forward(host(Xd), q(Wt), b, stride=s, pad=p, group=g, relu=True),
                    "fwd fp32")
    if "dx" in outs[1]:
        np.testing.assert_array_equal(outs[1]["dx"], host(dX32.to(torch.bfloat16)))
        assert_tc_close(host(dX32), oracle.conv_backward_data(host(dYd), q(Wt), X.shape, stride=s, pad=p, group=g),
                        "dgrad fp32")


@pytest.mark.parametrize("case", [(2, 3, 67, 67, 96, (11, 11), (4, 4), (0, 0), 1),
                                  (2, 96, 27, 27, 256, (5, 5), (1, 1), (2, 2), 2),
                                  CASES[7], (3, 64, 20, 20, 96, (3, 3), (1, 1), (1, 1), 1)],
                         ids=["conv1geom", "conv2geom", IDS[7], "C64O96"])
@pytest.mark.parametrize("sg", [0, 2])
def test_wgrad_reduce_rows_bit_identical(oracle, case, sg):
    """The per-(filter row, channel block) split reduction of the halo weight gradient
    (CAFFE_TUNE_WGRAD_REDUCE_ROWS, default off) gives the bits of the one-thread-per-weight reduction
    (and leaves the split-range form, CAFFE_TUNE_WGRAD_REDUCE_SG lowered to 2, and space-to-depth
    filters to it), with beta = 0 and 1 and the bias gradient from the ones chunk; and matches the
    oracle."""
    import torch
    import paper_1408_5093_b200 as cb
    from paper_1408_5093_b200 import _abi
    N, C, H, W, O, k, s, p, g = case
    X, Wt, b, dY = _inputs(case, 51)
    if C == 3:
        X = synth.int_pixels((N, C, H, W), 51)
    cl = torch.channels_last
    Xd = cuda(X).to(torch.bfloat16).contiguous(memory_format=cl)
    dYd = cuda(dY).to(torch.bfloat16).contiguous(memory_format=cl)
    prevW = cuda(synth.uniform(Wt.shape, 52, synth.S_AUX))
    prevb = cuda(synth.uniform((O,), 53, synth.S_AUX))
    outs = {}
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO, 2)
    if sg:
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_WGRAD_REDUCE_SG, sg)
    try:
        for rows in (0, 1):
            _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_WGRAD_REDUCE_ROWS, rows)
            dW, db = cb.conv_backward_weight(Xd, dYd, Wt.shape, stride=s, pad=p, group=g, math="bf16")
            dW1, db1 = cb.conv_backward_weight(Xd, dYd, Wt.shape, stride=s, pad=p, group=g, math="bf16", beta=1.0,
                                               dw=prevW.clone(), db=prevb.clone())
            outs[rows] = [host(t) for t in (dW, db, dW1, db1)]
    finally:
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_WGRAD_REDUCE_ROWS, 0)
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_WGRAD_REDUCE_SG, 0)
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO, 0)
    for a, b_ in zip(outs[0], outs[1]):
        np.testing.assert_array_equal(a, b_)
    rW, rb = oracle.conv_backward_weight(host(Xd), host(dYd), Wt.shape, stride=s, pad=p, group=g)
    assert_tc_close(outs[1][0], rW, "wgrad rows")
    assert_fp32_close(outs[1][1], rb, "bias grad rows")


@pytest.mark.parametrize("case,act,math,nhwc", [
    ((2, 128, 13, 13, 96, (3, 3), (1, 1), (1, 1), 1), "bf16", "bf16", True),    # im2col, TMA-store epilogue
    ((2, 64, 13, 13, 256, (3, 3), (1, 1), (1, 1), 2), "bf16", "bf16", True),    # grouped im2col (conv5-like)
    ((2, 96, 27, 27, 64, (5, 5), (1, 1), (2, 2), 2), "bf16", "bf16", True),     # halo tiles (generic epilogue)
    ((2, 8, 13, 13, 12, (3, 3), (1, 1), (1, 1), 2), "f32", "bf16", True),       # FP32 output, strided epilogue
    ((2, 3, 35, 35, 16, (11, 11), (4, 4), (0, 0), 1), "bf16", "bf16", True),    # space-to-depth: separate pass
    ((2, 8, 13, 13, 12, (3, 3), (1, 1), (1, 1), 2), "f32", "fp32", False),      # FP32 math, NCHW
], ids=["im2col", "grouped", "halo", "f32out", "s2d", "fp32math"])
def test_conv_backward_data_relu(oracle, case, act, math, nhwc):
    """caffe_conv_backward_data_relu (the data gradient through the ReLU that produced the layer's
    bottom, S:154 + S:208) gives exactly the bits of caffe_conv_backward_data followed by the ReLU
    backward, on every epilogue path; and the masked result matches the oracle."""
    import torch
    import paper_1408_5093_b200 as cb
    N, C, H, W, O, k, s, p, g = case
    X, Wt, b, dY = _inputs(case, 61)
    dt = torch.bfloat16 if act == "bf16" else torch.float32
    mf = torch.channels_last if nhwc else torch.contiguous_format
    top = cuda(X).to(dt).contiguous(memory_format=mf).relu_()     # ReLU output: zeros and positives
    dYd = cuda(dY).to(dt).contiguous(memory_format=mf)
    w = cuda(Wt)
    ref = torch.empty((N, C, H, W), device="cuda", dtype=dt).contiguous(memory_format=mf)
    cb.conv_backward_data(dYd, w, X.shape, stride=s, pad=p, group=g, math=math, out=ref)
    cb.relu_backward(top, ref, inplace=True)
    got = cb.conv_backward_data_relu(dYd, w, top, stride=s, pad=p, group=g, math=math)
    np.testing.assert_array_equal(host(got), host(ref))
    q = (lambda a: a) if math == "fp32" else oracle.quant_bf16
    want = oracle.conv_backward_data(q(host(dYd)), q(Wt), X.shape, stride=s, pad=p, group=g) * (host(top) > 0)
    if act == "bf16":
        assert_bf16_ulp(host(got), want, "masked dgrad (BF16 out)", atol=_atol(want))
    elif math == "fp32":
        assert_fp32_close(host(got), want, "masked dgrad fp32")
    else:
        assert_tc_close(host(got), want, "masked dgrad")
    # errors: shape and layout mismatches
    with pytest.raises(RuntimeError):
        cb.conv_backward_data_relu(dYd, w, top[:1], stride=s, pad=p, group=g, math=math)


@pytest.mark.parametrize("case", [CASES[7], CASES[1], (2, 64, 13, 13, 256, (3, 3), (1, 1), (1, 1), 2),
                                  (3, 40, 9, 11, 72, (5, 3), (1, 1), (2, 1), 1),
                                  (2, 96, 27, 27, 64, (5, 5), (1, 1), (2, 2), 2)],
                         ids=[IDS[7], IDS[1], "conv5geom", "k5x3", "conv2geom"])
@pytest.mark.parametrize("cta", [0, 1, 2])
def test_conv_stacked_halo(oracle, case, cta):
    """Stacked halo tiles (CAFFE_TUNE_HALO_STACKED=2: the images as one pixel sequence with shared
    zero rows/columns, 128-pixel tiles across image boundaries, one-row TMA boxes placed so every
    CTA's tile starts at the same shared-memory row) give oracle parity for the forward (bias, ReLU,
    FP32 and BF16 outputs) and the data gradient, single-CTA and CTA-pair, ragged last tile."""
    import torch
    import paper_1408_5093_b200 as cb
    from paper_1408_5093_b200 import _abi
    N, C, H, W, O, k, s, p, g = case
    X, Wt, b, dY = _inputs(case, 71)
    q = oracle.quant_bf16
    cl = torch.channels_last
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_STACKED, 2)
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_CTA_PAIR, cta)
    try:
        Xd = cuda(X).to(torch.bfloat16).contiguous(memory_format=cl)
        dYd = cuda(dY).to(torch.bfloat16).contiguous(memory_format=cl)
        Y = cb.conv_forward(Xd, cuda(Wt), cuda(b), stride=s, pad=p, group=g, relu=True, out_dtype=torch.float32)
        Y16 = cb.conv_forward(Xd, cuda(Wt), cuda(b), stride=s, pad=p, group=g, relu=True)
        dX = torch.empty((N, C, H, W), device="cuda").contiguous(memory_format=cl)
        cb.conv_backward_data(dYd, cuda(Wt), X.shape, stride=s, pad=p, group=g, out=dX)
        dX16 = torch.empty((N, C, H, W), device="cuda", dtype=torch.bfloat16).contiguous(memory_format=cl)
        cb.conv_backward_data(dYd, cuda(Wt), X.shape, stride=s, pad=p, group=g, out=dX16)
    finally:
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_STACKED, 1)
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_CTA_PAIR, 0)
    ry = oracle.conv_forward(host(Xd), q(Wt), b, stride=s, pad=p, group=g, relu=True)
    rx = oracle.conv_backward_data(host(dYd), q(Wt), X.shape, stride=s, pad=p, group=g)
    assert_tc_close(host(Y), ry, f"stacked fwd cta={cta}")
    assert_tc_close(host(dX), rx, f"stacked dgrad cta={cta}")
    np.testing.assert_array_equal(host(Y16), host(Y.to(torch.bfloat16)))
    np.testing.assert_array_equal(host(dX16), host(dX.to(torch.bfloat16)))


@pytest.mark.parametrize("case", [CASES[3], (2, 3, 67, 67, 96, (11, 11), (4, 4), (0, 0), 1),
                                  (2, 4, 9, 9, 8, (3, 3), (1, 1), (1, 1), 1)],
                         ids=["conv1like", "conv1geom", "plain3x3"])
@pytest.mark.parametrize("rows", [1, 2, 0])
def test_conv_i8_bottom(oracle, case, rows):
    """An int8 channels-last image batch (CAFFE_I8) packed by caffe_conv_pack_bottom gives the same
    bits as the same integers stored in BF16, for the prepacked forward and weight gradient
    (space-to-depth: the row-staged pack, CAFFE_TUNE_I8_ROWS=1, or the segment kernel; the
    element-form pack otherwise)."""
    import torch
    import paper_1408_5093_b200 as cb
    from paper_1408_5093_b200 import _abi
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_I8_ROWS, rows)
    try:
        _i8_bottom(oracle, case)
    finally:
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_I8_ROWS, 1)


def _i8_bottom(oracle, case):
    import torch
    import paper_1408_5093_b200 as cb
    N, C, H, W, O, k, s, p, g = case
    Xi = synth.int_pixels((N, C, H, W), 101)
    _, Wt, b, dY = _inputs(case, 101)
    cl = torch.channels_last
    w = cuda(Wt).to(torch.bfloat16)
    dYd = cuda(dY).to(torch.bfloat16).contiguous(memory_format=cl)
    outs = []
    for dt in (torch.bfloat16, torch.int8):
        x = cuda(Xi).to(dt).contiguous(memory_format=cl)
        ws = cb.conv_bottom_workspace(Xi.shape, Wt.shape, s, p, g, "bf16")
        cb.conv_pack_bottom(x, w, s, p, g, "bf16", ws=ws)
        y = cb.conv_forward(x, w, cuda(b), s, p, g, relu=True, ws=ws, prepacked=True, out_dtype=torch.float32)
        dW, db = cb.conv_backward_weight(x, dYd, Wt.shape, s, p, g, "bf16", ws=ws, prepacked=True)
        outs.append([host(t) for t in (y, dW, db)])
    for a, c in zip(*outs):
        np.testing.assert_array_equal(a, c)
    assert_tc_close(outs[1][0], oracle.conv_forward(Xi.astype(np.float64), oracle.quant_bf16(Wt), b, stride=s, pad=p,
                                                    group=g, relu=True), "i8 fwd")
    # an I8 bottom is refused where it is not packed
    import paper_1408_5093_b200._abi as abi
    with pytest.raises(abi.CaffeError):
        cb.conv_forward(cuda(Xi).to(torch.int8).contiguous(memory_format=cl), w, cuda(b), s, p, g)


@pytest.mark.parametrize("case", [CASES[3], CASES[7], (2, 96, 27, 27, 256, (5, 5), (1, 1), (2, 2), 2), CASES[1]],
                         ids=[IDS[3], IDS[7], "conv2geom", IDS[1]])
def test_conv_weights_prepacked(oracle, case):
    """caffe_conv_pack_weights + CAFFE_WEIGHTS_PREPACKED on a dedicated workspace gives the same bits
    as repacking the filter inside the forward / data-gradient call (im2col, halo, stacked and
    space-to-depth tiles)."""
    import torch
    import paper_1408_5093_b200 as cb
    N, C, H, W, O, k, s, p, g = case
    X, Wt, b, dY = _inputs(case, 121)
    cl = torch.channels_last
    Xd = cuda(X).to(torch.bfloat16).contiguous(memory_format=cl)
    dYd = cuda(dY).to(torch.bfloat16).contiguous(memory_format=cl)
    w = cuda(Wt).to(torch.bfloat16)
    wsf = cb.conv_workspace(X.shape, Wt.shape, s, p, g, "bf16", 0)
    wsd = cb.conv_workspace(X.shape, Wt.shape, s, p, g, "bf16", 1)
    cb.conv_pack_weights(w, X.shape, s, p, g, "bf16", 0, ws=wsf)
    cb.conv_pack_weights(w, X.shape, s, p, g, "bf16", 1, ws=wsd)
    y0 = cb.conv_forward(Xd, w, cuda(b), s, p, g, relu=True, out_dtype=torch.float32)
    y1 = cb.conv_forward(Xd, w, cuda(b), s, p, g, relu=True, out_dtype=torch.float32, ws=wsf, wprepacked=True)
    np.testing.assert_array_equal(host(y0), host(y1))
    dx0 = torch.empty((N, C, H, W), device="cuda").contiguous(memory_format=cl)
    dx1 = torch.empty((N, C, H, W), device="cuda").contiguous(memory_format=cl)
    cb.conv_backward_data(dYd, w, X.shape, s, p, g, out=dx0)
    cb.conv_backward_data(dYd, w, X.shape, s, p, g, out=dx1, ws=wsd, wprepacked=True)
    np.testing.assert_array_equal(host(dx0), host(dx1))
    with pytest.raises(RuntimeError):   # only the forward / data-gradient operands exist
        cb.conv_pack_weights(w, X.shape, s, p, g, "bf16", 2, ws=wsd)


CAP_CASES = [(3, 96, 27, 27, 256, (5, 5), (1, 1), (2, 2), 2),     # conv2 geometry: halo fwd / dgrad (N = 48)
             (2, 3, 67, 67, 96, (11, 11), (4, 4), (0, 0), 1),     # conv1 geometry: space-to-depth halo
             (3, 256, 13, 13, 384, (3, 3), (1, 1), (1, 1), 1),    # conv3 geometry: im2col tiles
             (3, 384, 13, 13, 256, (3, 3), (1, 1), (1, 1), 2),    # conv5 geometry: stacked halo forward
             CASES[1]]


@pytest.mark.parametrize("cap", [1, 2, 4])
@pytest.mark.parametrize("cta", [0, 1, 2])
@pytest.mark.parametrize("case", CAP_CASES, ids=["conv2geom", "conv1geom", "conv3geom", "conv5geom", IDS[1]])
def test_capped_grid_multi_unit(oracle, case, cta, cap):
    """CAFFE_TUNE_MAX_CTAS caps the persistent grid so every CTA (or CTA pair) loops over many work
    units -- the batch-256 schedule (12-24 units per pair: accumulator double buffers, TMEM slot
    reuse and mbarrier phases carried from unit to unit) at test sizes.  Results are bit-identical
    to the uncapped grid (work units and reduction orders do not depend on the grid) and match the
    oracle, for forward (BF16 and FP32 outputs), data and weight gradient, automatic and forced
    CTA-pair modes."""
    import torch
    import paper_1408_5093_b200 as cb
    from paper_1408_5093_b200 import _abi
    N, C, H, W, O, k, s, p, g = case
    X, Wt, b, dY = _inputs(case, 33)
    if C == 3:
        X = synth.int_pixels((N, C, H, W), 33)
    q = oracle.quant_bf16
    cl = torch.channels_last
    Xd = cuda(X).to(torch.bfloat16).contiguous(memory_format=cl)
    dYd = cuda(dY).to(torch.bfloat16).contiguous(memory_format=cl)
    outs = []
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_CTA_PAIR, cta)
    try:
        for mc in (0, cap):
            _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_MAX_CTAS, mc)
            r = {}
            r["y"] = cb.conv_forward(Xd, cuda(Wt), cuda(b), stride=s, pad=p, group=g, relu=True)
            r["y32"] = cb.conv_forward(Xd, cuda(Wt), cuda(b), stride=s, pad=p, group=g, relu=True,
                                       out_dtype=torch.float32)
            r["dw"], r["db"] = cb.conv_backward_weight(Xd, dYd, Wt.shape, stride=s, pad=p, group=g, math="bf16")
            if C != 3:
                dX = torch.empty((N, C, H, W), device="cuda").contiguous(memory_format=cl)
                cb.conv_backward_data(dYd, cuda(Wt), X.shape, stride=s, pad=p, group=g, out=dX)
                r["dx"] = dX
            torch.cuda.synchronize()
            outs.append({kk: host(v) for kk, v in r.items()})
    finally:
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_MAX_CTAS, 0)
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_CTA_PAIR, 0)
    for kk in outs[0]:
        np.testing.assert_array_equal(outs[0][kk], outs[1][kk], err_msg=f"{kk} capped at {cap} CTAs")
    got = outs[1]
    ry = oracle.conv_forward(host(Xd), q(Wt), b, stride=s, pad=p, group=g, relu=True)
    assert_tc_close(got["y32"], ry, "fwd capped")
    assert_bf16_ulp(got["y"], ry, "fwd capped (BF16 out)", atol=_atol(ry))
    rW, rb = oracle.conv_backward_weight(host(Xd), host(dYd), Wt.shape, stride=s, pad=p, group=g)
    assert_tc_close(got["dw"], rW, "wgrad capped")
    assert_fp32_close(got["db"], rb, "bias grad capped")
    if "dx" in got:
        assert_tc_close(got["dx"], oracle.conv_backward_data(host(dYd), q(Wt), X.shape, stride=s, pad=p, group=g),
                        "dgrad capped")


@pytest.mark.parametrize("cap", [1, 3])
@pytest.mark.parametrize("shape", [(256, 9216, 512), (256, 4096, 1000), (64, 800, 500)], ids=["fc6like", "fc8", "ip1"])
def test_capped_grid_inner_product(oracle, shape, cap):
    """Inner product (split-K forward / data gradient, CTA-pair weight gradient) on a capped grid:
    bit-identical to the full grid, and oracle parity."""
    import torch
    import paper_1408_5093_b200 as cb
    from paper_1408_5093_b200 import _abi
    N, K, O = shape
    x = cuda(synth.uniform((N, K), 34, synth.S_X)).to(torch.bfloat16)
    Wt = cuda(synth.xavier((O, K), 34)).to(torch.bfloat16)
    dy = cuda(synth.uniform((N, O), 34, synth.S_DY)).to(torch.bfloat16)
    outs = []
    try:
        for mc in (0, cap):
            _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_MAX_CTAS, mc)
            y = cb.ip_forward(x, Wt, None, out_dtype=torch.float32)
            dx = cb.ip_backward_data(dy, Wt, (N, K, 1, 1), out_dtype=torch.float32)
            dw, db = cb.ip_backward_weight(x, dy, (O, K))
            torch.cuda.synchronize()
            outs.append([host(t) for t in (y, dx, dw, db)])
    finally:
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_MAX_CTAS, 0)
    for a, c in zip(outs[0], outs[1]):
        np.testing.assert_array_equal(a, c)
    rdX, rdW, rdb = oracle.ip_backward(host(x), host(Wt), host(dy))
    assert_tc_close(outs[1][0], oracle.ip_forward(host(x), host(Wt)), "ip fwd capped")
    assert_tc_close(outs[1][1].reshape(N, K), rdX, "ip dgrad capped")
    assert_tc_close(outs[1][2], rdW, "ip wgrad capped")
    assert_tc_close(outs[1][3], rdb, "ip bias grad capped")


@pytest.mark.parametrize("case", [(2, 96, 27, 27, 256, (5, 5), (1, 1), (2, 2), 2),     # conv2: dgrad N = 48
                                  (2, 64, 20, 37, 48, (3, 3), (1, 1), (1, 1), 1),      # ragged tiles, 9 taps
                                  (2, 3, 67, 67, 96, (11, 11), (4, 4), (0, 0), 1)],   # conv1 geometry (s2d)
                         ids=["conv2geom", "H20W37", "conv1geom"])
def test_halo_btaps_bit_identical(oracle, case):
    """CAFFE_TUNE_HALO_BTAPS (5 taps' weight tiles per B pipeline stage in the compiled instance --
    conv2's 24-column data gradient -- or 1) gives the bits of one tap per stage (the MMA order is
    unchanged), for the halo forward and data gradient, CTA pairs and single CTAs."""
    import torch
    import paper_1408_5093_b200 as cb
    from paper_1408_5093_b200 import _abi
    N, C, H, W, O, k, s, p, g = case
    X, Wt, b, dY = _inputs(case, 51)
    if C == 3:
        X = synth.int_pixels((N, C, H, W), 51)
    cl = torch.channels_last
    Xd = cuda(X).to(torch.bfloat16).contiguous(memory_format=cl)
    dYd = cuda(dY).to(torch.bfloat16).contiguous(memory_format=cl)
    outs = {}
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO, 2)
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_JN, 0)   # the per-tap kernel's B stages
    try:
        for cta in (1, 2):
            _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_CTA_PAIR, cta)
            for bt in (1, 5):
                _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_BTAPS, bt)
                r = {"y": host(cb.conv_forward(Xd, cuda(Wt), cuda(b), stride=s, pad=p, group=g, relu=True))}
                if s[0] == 1:
                    dX = torch.empty((N, C, H, W), device="cuda", dtype=torch.bfloat16).contiguous(memory_format=cl)
                    cb.conv_backward_data(dYd, cuda(Wt), X.shape, stride=s, pad=p, group=g, out=dX)
                    r["dx"] = host(dX)
                outs[(cta, bt)] = r
    finally:
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_BTAPS, 0)
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_CTA_PAIR, 0)
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO, 0)
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_JN, 1)
    for (cta, bt), r in outs.items():
        for kk in r:
            np.testing.assert_array_equal(r[kk], outs[(cta, 1)][kk], err_msg=f"{kk} cta={cta} btaps={bt}")
    ry = oracle.conv_forward(host(Xd), oracle.quant_bf16(Wt), b, stride=s, pad=p, group=g, relu=True)
    assert_bf16_ulp(outs[(2, 5)]["y"], ry, "halo fwd btaps=5", atol=_atol(ry))


# data gradients of the column-taps-in-N kernel (A_HALO_JN): 5x5 filters with 48 channels per group
JN_CASES = [(2, 96, 27, 27, 256, (5, 5), (1, 1), (2, 2), 2),   # CaffeNet conv2: 240-column MMAs, 2 channel blocks
            (3, 96, 27, 27, 128, (5, 5), (1, 1), (2, 2), 2),   # one channel block, odd tile count
            (2, 48, 19, 27, 64, (5, 5), (1, 1), (2, 2), 1)]    # one group, ragged last tile (3 of 4 rows)
JN_IDS = ["conv2", "Og64", "g1H19"]


@pytest.mark.parametrize("max_ctas", [0, 4])
@pytest.mark.parametrize("case", JN_CASES, ids=JN_IDS)
def test_conv_dgrad_taps_in_n(oracle, case, max_ctas):
    """Data gradient with a filter row's taps in the MMA's N (CAFFE_TUNE_HALO_JN, the default for these
    shapes): BF16 channels-last result within 1 BF16 ulp of RNE(oracle) per element (R28) and rel-L2
    <= 1e-3; with the grid capped at 4 CTAs (2 pairs, one per group) every pair runs many tiles, so
    the accumulator double buffer, the A ring phases and the epilogue's cross-warp exchange buffers
    carry across units.  The per-tap kernel (CAFFE_TUNE_HALO_JN=0) agrees to FP32 summation order."""
    import torch
    import paper_1408_5093_b200 as cb
    from paper_1408_5093_b200 import _abi
    N, C, H, W, O, k, s, p, g = case
    X, Wt, b, dY = _inputs(case, 21)
    cl = torch.channels_last
    dYd = cuda(dY).to(torch.bfloat16).contiguous(memory_format=cl)
    ref = oracle.conv_backward_data(host(dYd), oracle.quant_bf16(Wt), X.shape, stride=s, pad=p, group=g)
    outs = {}
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_MAX_CTAS, max_ctas)
    try:
        for jn in (1, 0):
            _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_JN, jn)
            dX = torch.full((N, C, H, W), float("nan"), device="cuda", dtype=torch.bfloat16).contiguous(memory_format=cl)
            cb.conv_backward_data(dYd, cuda(Wt), X.shape, stride=s, pad=p, group=g, out=dX)
            outs[jn] = host(dX.float())
    finally:
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_JN, 1)
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_MAX_CTAS, 0)
    for jn, got in outs.items():
        assert np.isfinite(got).all(), f"jn={jn}: unwritten outputs"
        assert_bf16_ulp(got, ref, f"dgrad jn={jn} max_ctas={max_ctas}", atol=_atol(ref))
        assert_tc_close(got, oracle.quant_bf16(ref), f"dgrad jn={jn} max_ctas={max_ctas}")
    # different FP32 summation order: the two kernels really ran (not bit-identical)
    assert (outs[1] != outs[0]).any()


@pytest.mark.parametrize("case", [(2, 3, 227, 227, 96, (11, 11), (4, 4), (0, 0), 1),   # conv1: 28 tiles per image
                                  (2, 64, 24, 30, 96, (3, 3), (1, 1), (1, 1), 1),      # 6 tiles of 4 rows
                                  (3, 32, 16, 60, 64, (5, 5), (1, 1), (2, 2), 2)],     # 64-wide rows, 2 groups
                         ids=["conv1", "H24W30", "W60g2"])
@pytest.mark.parametrize("cta,max_ctas", [(2, 0), (2, 4), (1, 3)])
def test_halo_merged_window_bit_identical(oracle, case, cta, max_ctas):
    """CAFFE_TUNE_HALO_MERGE (off by default: a CTA's two accumulators take consecutive row blocks of
    one image and share one staged window, three stages deep) writes exactly the bits of one window per tile, for
    the halo forward (bias + ReLU, BF16 channels-last) and the stride-1 data gradient, CTA pairs and
    single CTAs, full and capped grids (many units per CTA); the result meets the oracle bar."""
    import torch
    import paper_1408_5093_b200 as cb
    from paper_1408_5093_b200 import _abi
    N, C, H, W, O, k, s, p, g = case
    X, Wt, b, dY = _inputs(case, 61)
    if C == 3:
        X = synth.int_pixels((N, C, H, W), 61)
    cl = torch.channels_last
    Xd = cuda(X).to(torch.bfloat16).contiguous(memory_format=cl)
    dYd = cuda(dY).to(torch.bfloat16).contiguous(memory_format=cl)
    outs = {}
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO, 2)
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_CTA_PAIR, cta)
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_MAX_CTAS, max_ctas)
    try:
        for merge in (1, 0):
            _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_MERGE, merge)
            r = {"y": host(cb.conv_forward(Xd, cuda(Wt), cuda(b), stride=s, pad=p, group=g, relu=True))}
            if s[0] == 1:
                dX = torch.empty((N, C, H, W), device="cuda", dtype=torch.bfloat16).contiguous(memory_format=cl)
                cb.conv_backward_data(dYd, cuda(Wt), X.shape, stride=s, pad=p, group=g, out=dX)
                r["dx"] = host(dX)
            outs[merge] = r
    finally:
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_MERGE, 0)
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_MAX_CTAS, 0)
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_CTA_PAIR, 0)
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO, 0)
    for kk in outs[0]:
        np.testing.assert_array_equal(outs[1][kk], outs[0][kk], err_msg=f"{kk} merged vs per-tile windows")
    ry = oracle.conv_forward(host(Xd), oracle.quant_bf16(Wt), b, stride=s, pad=p, group=g, relu=True)
    assert_bf16_ulp(outs[1]["y"], ry, "halo fwd merged", atol=_atol(ry))
    if "dx" in outs[1]:
        rd = oracle.conv_backward_data(host(dYd), oracle.quant_bf16(Wt), X.shape, stride=s, pad=p, group=g)
        assert_bf16_ulp(outs[1]["dx"], rd, "halo dgrad merged", atol=_atol(rd))
