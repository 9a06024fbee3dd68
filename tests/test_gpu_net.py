"""Net-level parity (-m gpu): the straight-line LeNet / CaffeNet training step run through the C ABI
(paper_1408_5093_b200.nets) against the oracle on the same seeded inputs and weights.

* end to end: the loss of the GPU step matches oracle/net.py's forward to 1e-3 relative
  (SURVEY 8(c) "Nets"), with BF16 GEMM operands on both sides;
* teacher-forced: every layer's forward output and every parameter / data gradient is compared with
  the oracle layer applied to the GPU's OWN inputs (its stored activation and the top diff that
  layer consumed).  Max-pool and ReLU discontinuities make a free-running comparison of gradients
  meaningless (a 1-ulp difference flips an argmax), so the chain is checked link by link.
  Tolerances: the per-layer bars (rel-L2 1e-3 for tensor-core passes; BF16-stored results are
  compared after rounding the oracle's value to BF16 the same way).
"""
import numpy as np
import pytest

import synth
from _helpers import assert_tc_close, host

pytestmark = pytest.mark.gpu

LRN = dict(size=5, alpha=1e-4, beta=0.75, k=1.0)


def _build(which, batch, act, fc_hwc=False):
    import torch
    from paper_1408_5093_b200 import nets
    layers, shape = (nets.LENET, nets.LENET_INPUT) if which == "lenet" else (nets.CAFFENET, nets.CAFFENET_INPUT)
    dt = torch.float32 if act == "f32" else torch.bfloat16
    saved = nets.Net.fc_hwc
    nets.Net.fc_hwc = fc_hwc   # read at construction (weight layout of the first inner product)
    try:
        net = nets.Net(layers, batch, shape, torch.device("cuda"), act_dtype=dt, math="bf16", seed=0)
    finally:
        nets.Net.fc_hwc = saved
    assert bool(net.hwc) == fc_hwc
    net.fuse_pool_lrn = False   # every layer's blobs stored (the fused kernels: test_fused_pool_lrn_bit_identical)
    X = synth.int_pixels((batch,) + tuple(shape), 7) if which == "caffenet" else \
        synth.mnist_pixels((batch,) + tuple(shape), 7)
    lab = synth.labels(batch, net.shapes[-1][1], 7)
    net.a[0].copy_(torch.from_numpy(X))
    net.labels.copy_(torch.from_numpy(lab))
    net.grads.zero_()
    net.forward()
    net.backward()
    torch.cuda.synchronize()
    return net, X, lab


def _stored(net, ref, i_out):
    """Round an oracle result the way the GPU stored blob i_out is stored (BF16 activations)."""
    import torch
    import oracle
    t = net.a[i_out] if i_out < len(net.a) else None
    if t is not None and t.dtype == torch.bfloat16:
        return oracle.quant_bf16(np.asarray(ref, np.float32))
    return ref


@pytest.mark.parametrize("which,batch,act,hwc", [("lenet", 16, "f32", False), ("lenet", 16, "bf16", False),
                                                 ("caffenet", 2, "f32", False), ("caffenet", 2, "bf16", False),
                                                 ("lenet", 16, "bf16", True), ("caffenet", 2, "bf16", True)])
def test_net_teacher_forced(oracle, which, batch, act, hwc):
    """(hwc: the first inner product's weight columns stored in the (h, w, c) order of its channels-last
    input, Net.fc_hwc -- compared through Net.canonical in the (c, h, w) order of S:130.)"""
    from oracle import net as onet
    net, X, lab = _build(which, batch, act, fc_hwc=hwc)
    q = oracle.quant_bf16
    n = len(net.layers)
    # ---------------- end-to-end loss vs the oracle's own forward (BF16 GEMM operands)
    olayers = onet.LENET if which == "lenet" else onet.CAFFENET
    params = {net.layers[i].name: (net.canonical(i, host(net.W[i])).astype(np.float64), host(net.B[i]).astype(np.float64))
              for (i, _, _) in net.pspecs}
    oloss, _, _ = onet.forward_backward(olayers, X, params, lab, quant=q)
    assert abs(float(net.loss) - oloss) <= 1e-3 * abs(oloss), (float(net.loss), oloss)
    # ---------------- forward, layer by layer on the GPU's own inputs
    for i, L in enumerate(net.layers[:-1]):
        x = host(net.a[i]).astype(np.float64)
        last = i + 1 == n - 1
        y = host(net.scores if last else net.a[i + 1])
        W = net.canonical(i, host(net.W[i])) if i in net.W else None
        if L.kind == "conv":
            ref = oracle.conv_forward(q(x), q(W), host(net.B[i]), stride=(L.stride,) * 2, pad=(L.pad,) * 2,
                                      group=L.group, relu=L.relu)
        elif L.kind == "pool":
            ref = oracle.maxpool_forward(x.astype(np.float32), (L.kernel,) * 2, (L.stride,) * 2)[0]
            np.testing.assert_array_equal(y, ref.reshape(y.shape))
            continue
        elif L.kind == "lrn":
            ref = oracle.lrn_forward(x, **LRN)
        else:
            ref = oracle.ip_forward(q(x), q(W), host(net.B[i]))
            if L.relu:
                ref = np.maximum(ref, 0)
        ref = ref.reshape(y.shape)
        assert_tc_close(y, ref if last else _stored(net, ref, i + 1), f"{which} {L.name} fwd")
    # ---------------- softmax-loss gradient on the GPU's scores
    lo, dref = oracle.softmax_loss(host(net.scores), lab)
    assert abs(float(net.loss) - lo) <= 1e-5 * (abs(lo) + 1)
    # ---------------- backward, layer by layer on the GPU's own (x, consumed dy)
    for i in range(n - 2, -1, -1):
        L = net.layers[i]
        x = host(net.a[i]).astype(np.float64)
        dy = host(net.dscores if i + 1 == n - 1 else net.d[i + 1]).astype(np.float64)  # after in-place ReLU mask
        mask_in = None
        if i > 0 and net.layers[i - 1].kind in ("conv", "ip") and net.layers[i - 1].relu:
            mask_in = x > 0            # d[i] was masked in place by the layer below's ReLU backward
        if L.kind == "conv":
            W = host(net.W[i])
            dW, db = oracle.conv_backward_weight(q(x), q(dy), W.shape, stride=(L.stride,) * 2, pad=(L.pad,) * 2,
                                                 group=L.group)
            assert_tc_close(host(net.dW[i]), dW, f"{which} {L.name} dW")
            assert_tc_close(host(net.dB[i]), dy.sum(axis=(0, 2, 3)), f"{which} {L.name} db")
            if i == 0:
                continue
            ref = oracle.conv_backward_data(q(dy), q(W), x.shape, stride=(L.stride,) * 2, pad=(L.pad,) * 2,
                                            group=L.group)
        elif L.kind == "ip":
            W = net.canonical(i, host(net.W[i]))
            dX, dW, _ = oracle.ip_backward(q(x), q(W), q(dy.reshape(dy.shape[0], -1)))
            assert_tc_close(net.canonical(i, host(net.dW[i])), dW, f"{which} {L.name} dW")
            assert_tc_close(host(net.dB[i]), dy.reshape(dy.shape[0], -1).sum(0), f"{which} {L.name} db")
            ref = dX.reshape(x.shape)
        elif L.kind == "pool":
            _, m = oracle.maxpool_forward(x.astype(np.float32), (L.kernel,) * 2, (L.stride,) * 2)
            ref = oracle.maxpool_backward(dy.astype(np.float32), m, x.shape, (L.kernel,) * 2, (L.stride,) * 2)
        else:  # lrn
            ref = oracle.lrn_backward(x, dy, **LRN)
        if mask_in is not None:
            ref = np.where(mask_in, ref, 0.0)
        got = host(net.d[i])
        ref = _stored(net, ref, i)
        if L.kind == "pool" and act == "f32":
            np.testing.assert_array_equal(got, ref)
        else:
            assert_tc_close(got, ref, f"{which} {L.name} dX")
    assert np.isfinite(float(net.loss))


@pytest.mark.parametrize("fuse", [False, True])
def test_overlapped_update_matches_serial(fuse):
    """Net.step(overlap_update=True) (per-layer SGD on a side stream, weight gradients on their own
    stream; with fuse, the inner-product updates fused into their weight-gradient GEMMs where the
    fan-in allows -- LeNet ip1) gives the same parameters, bit for bit, as the single update after
    the backward pass."""
    import torch
    import synth
    from paper_1408_5093_b200 import nets
    dev = torch.device("cuda")
    outs = []
    for overlap in (False, True):
        net = nets.Net(nets.LENET, 16, nets.LENET_INPUT, dev, math="bf16", seed=3)
        net.fuse_ip_sgd = fuse
        net.a[0].copy_(torch.from_numpy(synth.mnist_pixels((16,) + tuple(nets.LENET_INPUT), 3)).to(torch.bfloat16))
        net.labels.copy_(torch.from_numpy(synth.labels(16, 10, 3)))
        for _ in range(2):
            net.step(overlap_update=overlap)
        torch.cuda.synchronize()
        outs.append((net.params.cpu().numpy().copy(), net.params_bf16.float().cpu().numpy().copy()))
    import numpy as np
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])


def test_int8_input_batch_matches_bf16():
    """Net(input_i8=True) (integer image batch stored as int8, converted by conv1's pack) trains to
    the same parameters, bit for bit, as the same integers stored in BF16."""
    import torch
    import synth
    from paper_1408_5093_b200 import nets
    dev = torch.device("cuda")
    B = 4
    X = synth.int_pixels((B,) + tuple(nets.CAFFENET_INPUT), 7)
    outs = []
    for i8 in (False, True):
        net = nets.Net(nets.CAFFENET, B, nets.CAFFENET_INPUT, dev, math="bf16", seed=5, input_i8=i8)
        assert net.input_i8 == i8
        net.a[0].copy_(torch.from_numpy(X).to(net.a[0].dtype))
        net.labels.copy_(torch.from_numpy(synth.labels(B, 1000, 7)))
        for _ in range(2):
            net.step()
        torch.cuda.synchronize()
        outs.append(net.params.cpu().numpy().copy())
    import numpy as np
    np.testing.assert_array_equal(outs[0], outs[1])


def test_prepacked_weights_step_matches():
    """Net.prepack_weights (conv weight operands repacked after each update into per-layer
    workspaces, CAFFE_WEIGHTS_PREPACKED in the passes) trains to the same parameters, bit for bit."""
    import torch
    import synth
    from paper_1408_5093_b200 import nets
    dev = torch.device("cuda")
    B = 4
    X = synth.int_pixels((B,) + tuple(nets.CAFFENET_INPUT), 9)
    outs = []
    for pre in (False, True):
        old = nets.Net.prepack_weights
        nets.Net.prepack_weights = pre
        try:
            net = nets.Net(nets.CAFFENET, B, nets.CAFFENET_INPUT, dev, math="bf16", seed=6)
        finally:
            nets.Net.prepack_weights = old
        assert bool(net.wsf) == pre
        net.a[0].copy_(torch.from_numpy(X).to(net.a[0].dtype))
        net.labels.copy_(torch.from_numpy(synth.labels(B, 1000, 9)))
        for _ in range(2):
            net.step()
        torch.cuda.synchronize()
        outs.append(net.params.cpu().numpy().copy())
    import numpy as np
    np.testing.assert_array_equal(outs[0], outs[1])


def test_dp_path_single_rank_nccl():
    """The data-parallel step (bucketed NCCL all-reduce hooks, finish, update with 1/W) run as a
    one-rank NCCL group equals the serial single-GPU step bit for bit (the sum over one rank is the
    identity): covers the W > 1 code path on one GPU."""
    import os
    import torch
    import torch.distributed as dist
    import synth
    from paper_1408_5093_b200 import nets
    from paper_1408_5093_b200.dp import GradAllReduce
    dev = torch.device("cuda")
    dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29533", rank=0, world_size=1)
    try:
        outs = []
        for dp in (False, True):
            net = nets.Net(nets.LENET, 16, nets.LENET_INPUT, dev, math="bf16", seed=4)
            net.a[0].copy_(torch.from_numpy(synth.mnist_pixels((16,) + tuple(nets.LENET_INPUT), 4)).to(torch.bfloat16))
            net.labels.copy_(torch.from_numpy(synth.labels(16, 10, 4)))
            ar = GradAllReduce(net.grads, net.segments, 1, bucket_bytes=64 << 10) if dp else None
            for _ in range(2):
                if dp:
                    net.step(ar)
                else:
                    net.step(overlap_update=False)
            torch.cuda.synchronize()
            outs.append(net.params.cpu().numpy().copy())
        import numpy as np
        np.testing.assert_array_equal(outs[0], outs[1])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", [1, 2])
def test_side_stream_weight_packs_bit_identical(mode):
    """Net.pack_side (conv weight operands packed at the start of the step on a side stream into
    dedicated workspaces; 1: forward, 2: forward + data gradient) gives exactly the bits of the
    per-call repacks: loss, every parameter gradient and the updated parameters after two steps."""
    import torch
    from paper_1408_5093_b200 import nets
    outs = []
    for ps in (0, mode):
        net = nets.Net(nets.CAFFENET, 4, nets.CAFFENET_INPUT, torch.device("cuda"), math="bf16", seed=0)
        net.pack_side = ps
        net.a[0].copy_(torch.from_numpy(synth.int_pixels((4,) + tuple(nets.CAFFENET_INPUT), 5)))
        net.labels.copy_(torch.from_numpy(synth.labels(4, 1000, 5)))
        for _ in range(2):
            net.step()
        torch.cuda.synchronize()
        outs.append((float(net.loss), net.grads.cpu().numpy().copy(), net.params.cpu().numpy().copy()))
    assert outs[0][0] == outs[1][0]
    np.testing.assert_array_equal(outs[0][1], outs[1][1])
    np.testing.assert_array_equal(outs[0][2], outs[1][2])


def test_pdl_launches_bit_identical():
    """CAFFE_TUNE_PDL (tensor-core GEMMs launched with programmatic stream serialization; each waits
    on griddepcontrol.wait before touching global memory) gives exactly the bits of ordinary stream
    order: two eager steps and two graph replays of the CaffeNet step (batch 4, three streams)."""
    import torch
    from paper_1408_5093_b200 import _abi, nets
    outs = []
    try:
        for pdl in (0, 1):
            _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_PDL, pdl)
            net = nets.Net(nets.CAFFENET, 4, nets.CAFFENET_INPUT, torch.device("cuda"), math="bf16", seed=0,
                           input_i8=True)
            net.a[0].copy_(torch.from_numpy(synth.int_pixels((4,) + tuple(nets.CAFFENET_INPUT), 9)).to(torch.int8))
            net.labels.copy_(torch.from_numpy(synth.labels(4, 1000, 9)))
            for _ in range(2):
                net.step()
            g = net.capture()
            for _ in range(2):
                g.replay()
            torch.cuda.synchronize()
            outs.append((float(net.loss), net.grads.cpu().numpy().copy(), net.params.cpu().numpy().copy()))
    finally:
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_PDL, 0)
    assert outs[0][0] == outs[1][0]
    np.testing.assert_array_equal(outs[0][1], outs[1][1])
    np.testing.assert_array_equal(outs[0][2], outs[1][2])
